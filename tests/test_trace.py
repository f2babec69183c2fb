"""Trace output: gpk_write_trace_csv reproduces
the reference's CSV (proj/core/src/trace.cpp:7-44): header, column order and
shortest round-trip doubles. Host-only, so it runs on CPU."""
import numpy as np


def format_double(v):  # trace.cpp:7-18
    for prec in (15, 16, 17):
        s = "%.*g" % (prec, v)
        if float(s) == v:
            return s
    return "%.17g" % v


def test_trace_csv_matches_reference_format(tmp_path):
    import paper_2405_18457_b200 as G
    d = 2
    rng = np.random.default_rng(0)
    rows = 3
    tr = {"constrained": rng.random((rows, d + 2)) + 0.5, "gradient": rng.standard_normal((rows, d + 2)),
          "mean_residual_norm": rng.random(rows) * 1e-2, "probe_residual_norm": rng.random(rows) * 1e-2,
          "epochs": np.array([3.0, 2.5, 1.0 / 3.0]), "grad_inf_norm": rng.random(rows),
          "iterations": np.array([3, 2, 1]), "solver_diverged": np.array([False, True, False]),
          "step_seconds": np.array([0.1, 0.2, 0.3]), "solver_seconds": np.array([0.05, 0.1, 0.15])}
    path = tmp_path / "trace.csv"
    G.gpiter.write_trace_csv(path, tr, d)
    lines = path.read_text().splitlines()
    assert lines[0] == ("step,lengthscale_0,lengthscale_1,signal_scale,noise_scale,mean_residual_norm,"
                        "probe_residual_norm,epochs,solver_seconds_cum,total_seconds_cum,test_rmse,test_llh,"
                        "grad_inf_norm,diverged")
    scum = np.cumsum(tr["solver_seconds"])
    tcum = np.cumsum(tr["step_seconds"])
    for t in range(rows):
        want = [str(t)] + [format_double(v) for v in tr["constrained"][t]]
        want += [format_double(tr[k][t]) for k in ("mean_residual_norm", "probe_residual_norm", "epochs")]
        want += [format_double(scum[t]), format_double(tcum[t]), "", "", format_double(tr["grad_inf_norm"][t]),
                 "1" if tr["solver_diverged"][t] else "0"]
        assert lines[t + 1] == ",".join(want)
        assert [float(x) for x in lines[t + 1].split(",")[1:d + 3]] == list(tr["constrained"][t])  # round trip


def test_compare_oracle_files_match_reference_format(tmp_path):
    """differences.csv / compare_oracle.json of `gpiter compare-oracle`
    (proj/tools/gpiter_cli.cpp:247-278): header, round-trip doubles, log10 bins."""
    from paper_2405_18457_b200 import outputs
    a = np.array([[1.0, 0.5, 0.25], [1.1, 0.6, 0.3]])
    b = a + np.array([[0.0, 3e-9, 2e-5], [0.5, 1e-3, 4.0]])
    out = outputs.write_differences(tmp_path, a, b)
    lines = (tmp_path / "differences.csv").read_text().splitlines()
    assert lines[0] == "step,coordinate,iterative,exact,abs_diff"
    assert len(lines) == 1 + a.size
    assert lines[1] == "0,0,1,1,0"
    t, k, it, ex, df = lines[3].split(",")
    assert (t, k) == ("0", "2") and float(it) == a[0, 2] and float(ex) == b[0, 2] and float(df) == abs(a[0, 2] - b[0, 2])
    assert out["histogram_bin_edges"][0] == "<=1e-8" and len(out["histogram_counts"]) == 10
    # 0 and 3e-9 -> bin 0; 2e-5 -> 1e-5..1e-4 (4); 0.5 -> 1e-1..1 (8); 1e-3 -> 1e-3..1e-2 (6); 4 -> >1 (9)
    assert out["histogram_counts"] == [2, 0, 0, 0, 1, 0, 1, 0, 1, 1]
    assert out["max_abs_diff"] == 4.0


def test_summary_json_fields(tmp_path):
    """summary.json of `gpiter train` (gpiter_cli.cpp:118-143) for a trace."""
    import json

    from paper_2405_18457_b200 import gpiter, outputs
    res = {"final_raw": np.array([gpiter.softplus_inverse(v) for v in (0.7, 1.3, 0.9, 0.2)]),
           "epochs": np.array([3.0, 2.5]), "solver_diverged": np.array([False, True]),
           "solver_seconds": np.array([0.1, 0.2]), "step_seconds": np.array([0.3, 0.4]),
           "constrained": np.ones((2, 4))}
    cfg = gpiter.OuterConfig(solver=gpiter.SolverConfig(kind=1), steps=2)
    s = outputs.write_summary(tmp_path / "summary.json", res, cfg, n_train=100)
    back = json.loads((tmp_path / "summary.json").read_text())
    assert back == s
    assert s["schema_version"] == 1 and s["steps_completed"] == 2 and s["diverged_steps"] == 1
    assert abs(s["total_epochs"] - 5.5) < 1e-15 and s["config"]["solver"] == "ap"
    assert np.allclose(s["hyperparameters"]["lengthscales"], [0.7, 1.3])
    assert abs(s["solver_seconds"] - 0.3) < 1e-15 and abs(s["total_seconds"] - 0.7) < 1e-15
