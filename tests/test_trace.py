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
