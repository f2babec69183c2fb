"""Multi-GPU decomposition, checked on CPU with a world-size-2 gloo group.

The library's multi-GPU mode (csrc/gpk_api.cu, sharded operator) splits the
rows into 32-aligned shards (gpk_shard_rows), all-gathers the search
direction in FP32 (each rank then builds the operator's TF32 images itself),
all-gathers per-rank column partial sums and adds them in rank order, splits
the gradient pass's symmetric tile list evenly across ranks, and for SGD
all-reduces one buffer of minibatch partial products per iteration.
Here two gloo processes run exactly that decomposition with the FP64 oracle
doing each rank's local work, and must reproduce the single-process oracle:
CG iteration counts equal, solutions and gradient forms to ~1e-10.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(n=200, d=3, s=3):
    rng = np.random.default_rng(5)
    X = np.asfortranarray(rng.standard_normal((n, d)))
    T = np.asfortranarray(rng.standard_normal((n, s + 1)))
    Z = np.asfortranarray(rng.standard_normal((n, s)))
    return X, T, Z


def _gather_rows(dist, local, S, world):
    """All-gather equal (S-row, zero-padded) shards -> full array (rows beyond n dropped by caller)."""
    import torch
    pad = np.zeros((S, local.shape[1]))
    pad[: local.shape[0]] = local
    t = torch.from_numpy(pad)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return np.concatenate([o.numpy() for o in out], axis=0)


def _sum_in_rank_order(dist, vec, world):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(vec, dtype=np.float64))
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    acc = np.zeros_like(vec, dtype=np.float64)
    for o in out:  # fixed rank order: every rank takes identical decisions
        acc = acc + o.numpy()
    return acc


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2405_18457_b200 import parallel as P

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    X, T, Z = _problem()
    n, d = X.shape
    m = T.shape[1]
    raw = O.raw_from_constrained([0.9, 1.1, 1.3, 1.0, 0.5])
    S = P.shard_stride(n, world)
    r0, r1 = P.shard_rows(n, world, rank)
    rows = np.arange(r0, r1, dtype=np.int32)

    def apply_local(v_loc):
        """apply_local_ring (csrc/gpk_api.cu): the FP32 direction travels one hop
        per step around the ring (send slice rk - j to rk + 1, receive slice
        rk - j - 1 from rk - 1) and the product accumulates slice by slice,
        own slice first."""
        import torch
        slices = {rank: np.zeros((S, m), dtype=np.float32)}
        slices[rank][: v_loc.shape[0]] = v_loc.astype(np.float32)
        nxt, prv = (rank + 1) % world, (rank - 1) % world
        for j in range(world - 1):
            snd, rcv = (rank - j) % world, (rank - j - 1) % world
            buf = torch.zeros((S, m), dtype=torch.float32)
            if rank % 2 == 0:  # pair the blocking calls
                dist.send(torch.from_numpy(slices[snd]), nxt)
                dist.recv(buf, prv)
            else:
                dist.recv(buf, prv)
                dist.send(torch.from_numpy(slices[snd]), nxt)
            slices[rcv] = buf.numpy()
        out = np.zeros((len(rows), m))
        for j in range(world):
            src = (rank - j) % world
            c0, c1 = src * S, min(n, (src + 1) * S)
            if c1 <= c0:
                continue
            v_full = np.zeros((n, m))
            v_full[c0:c1] = slices[src][: c1 - c0]
            out = out + O.apply_rows(X, raw, rows, np.asfortranarray(v_full))
        return out

    def colsum(a, b=None):
        return (a * (a if b is None else b)).sum(axis=0)

    # ---- sharded CG (solvers.cpp:34-88 without preconditioner) ----
    tol, max_epochs = 1e-4, 200  # the direction crosses ranks in FP32: 1e-6 is below what it carries
    scales = np.sqrt(_sum_in_rank_order(dist, colsum(T[r0:r1]), world)) + 1e-12
    V = np.zeros((r1 - r0, m))
    R = T[r0:r1] - apply_local(V)
    p = R.copy()
    dvec = p.copy()
    gamma = _sum_in_rank_order(dist, colsum(R, p), world)

    def done():
        ss = _sum_in_rank_order(dist, colsum(R), world)
        mean = np.sqrt(ss[0]) / scales[0]
        probe = np.mean(np.sqrt(ss[1:]) / scales[1:])
        return mean <= tol and probe <= tol

    t = 0
    while t < max_epochs and not done():
        hd = apply_local(dvec)
        denom = _sum_in_rank_order(dist, colsum(dvec, hd), world)
        alpha = gamma / denom
        V = V + dvec * alpha
        R = R - hd * alpha
        p = R.copy()
        gnext = _sum_in_rank_order(dist, colsum(R, p), world)
        beta = np.where(gamma != 0.0, gnext / np.where(gamma != 0.0, gamma, 1.0), 0.0)
        gamma = gnext
        dvec = p + dvec * beta
        t += 1
    V_full = _gather_rows(dist, V, S, world)[:n]

    # ---- sharded gradient pass: symmetric tile list split across ranks ----
    ls = np.array([O.softplus(x) for x in raw[:d]])
    sig = O.softplus(raw[d])
    xs = X / ls
    tb, te = P.grad_tile_range(n, world, rank, symmetric=True)
    part = np.zeros(d + 1)  # [lengthscale sums..., signal sum]
    for L in range(tb, te):
        ti, tc = P.tile_coords(L, n, symmetric=True)
        w = 2.0 if tc != ti else 1.0
        i = np.arange(ti * P.TILE, min(n, (ti + 1) * P.TILE))
        c = np.arange(tc * P.TILE, min(n, (tc + 1) * P.TILE))
        diff = xs[c][None, :, :] - xs[i][:, None, :]
        r = np.sqrt((diff ** 2).sum(-1))
        e0 = np.exp(-np.sqrt(3) * r)
        kv = (1 + np.sqrt(3) * r) * e0
        g = Z[i] @ Z[c].T
        part[d] += w * (kv * g).sum()
        part[:d] += w * np.einsum("ic,icq->q", e0 * g, diff ** 2)
    tot = _sum_in_rank_order(dist, part, world)
    forms = np.empty(d + 2)
    forms[:d] = (1.0 / ls) * 3.0 * sig ** 2 * tot[:d]
    forms[d] = (2.0 / sig) * sig ** 2 * tot[d]
    forms[d + 1] = 2.0 * O.softplus(raw[d + 1]) * _sum_in_rank_order(dist, np.array([(Z[r0:r1] ** 2).sum()]), world)[0]
    q.put((rank, t, V_full, forms, (r0, r1)))
    dist.destroy_process_group()


def _sgd_worker(rank, world, port, q, cfg):
    """Row-sharded SGD exactly as solve_sgd_lazy (csrc/gpk_api.cu,
    csrc/sgd_lazy.cu) decomposes it: momentum evaluated lazily from each row's
    last update (tables P = rho^Delta, S = rho + .. + rho^Delta), the minibatch
    rows contracted against this rank's own rows at their current V(t), the
    owning rank folding in -B[idx] (and H's noise diagonal) plus the old
    residual squares of its rows, one all-reduce (sum) of that buffer per
    iteration, each rank updating only its own minibatch rows."""
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2405_18457_b200 import parallel as P

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    X, T, _ = _problem()
    n, m = X.shape[0], T.shape[1]
    raw = O.raw_from_constrained([0.9, 1.1, 1.3, 1.0, 0.5])
    H = O.dense(X, raw)
    S = P.shard_stride(n, world)
    r0, r1 = P.shard_rows(n, world, rank)
    b = min(cfg["batch_size"], n)
    budget = int(np.ceil(cfg["max_epochs"] * n / b))
    step = cfg["learning_rate"] / b
    rho = cfg["momentum"]
    Pt, St = [1.0], [0.0]
    for _ in range(budget):
        Pt.append(Pt[-1] * rho)
        St.append(St[-1] + Pt[-1])
    Pt, St = np.array(Pt), np.array(St)
    batches = O.sample_without_replacement(cfg["seed"], 6, cfg["substream"], n, b, budget)
    scales = np.sqrt(_sum_in_rank_order(dist, (T[r0:r1] ** 2).sum(0), world)) + 1e-12
    Vb = np.zeros((r1 - r0, m))
    Mb = np.zeros_like(Vb)
    tau = np.full(r1 - r0, -1)
    R = T[r0:r1].copy()
    sumsq = _sum_in_rank_order(dist, (R ** 2).sum(0), world)

    def done(ss):
        ss = np.maximum(ss, 0.0)
        return np.sqrt(ss[0]) / scales[0] <= cfg["tolerance"] and \
            np.mean(np.sqrt(ss[1:]) / scales[1:]) <= cfg["tolerance"]

    def delta(t):
        return np.clip(t - tau - 1, 0, budget)

    t = 0
    finished = done(sumsq)
    while not finished and t < budget:
        idx = batches[t]
        own = (idx >= r0) & (idx < r1)
        vt = Vb + St[delta(t)][:, None] * Mb
        part = H[idx][:, r0:r1] @ vt
        part[own] -= T[idx[own]]
        old = (R[idx[own] - r0] ** 2).sum(0)
        buf = torch.from_numpy(np.concatenate([part.ravel(), old, [0.0]]))
        dist.all_reduce(buf)
        g = buf.numpy()[: b * m].reshape(b, m)
        sumsq = sumsq + ((g ** 2).sum(0) - buf.numpy()[b * m: b * m + m])
        li = idx[own] - r0
        dl = delta(t)[li]
        mt = Pt[dl][:, None] * Mb[li]
        mn = mt * rho - step * g[own]
        Vb[li] = vt[li] + mn
        Mb[li] = mn
        tau[li] = t
        R[li] = -g[own]
        t += 1
        finished = done(sumsq)
    V = Vb + St[delta(t)][:, None] * Mb
    q.put((rank, t, _gather_rows(dist, V, S, world)[:n]))
    dist.destroy_process_group()


def test_world2_gloo_sharded_sgd_matches_single_process(oracle):
    import torch.multiprocessing as mp
    cfg = dict(kind=2, tolerance=0.05, max_epochs=30, batch_size=24, learning_rate=1.0, momentum=0.9, seed=4,
               substream=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sgd_worker, args=(r, 2, port, q, cfg)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, t0, V0), (_, t1, V1) = res
    assert t0 == t1 and np.array_equal(V0, V1)
    X, T, _ = _problem()
    raw = oracle.raw_from_constrained([0.9, 1.1, 1.3, 1.0, 0.5])
    ref = oracle.solve(X, raw, T, oracle.solver_config(**{k: v for k, v in cfg.items()}))
    assert abs(ref["iterations"] - t0) <= 1
    if ref["iterations"] == t0:
        assert np.max(np.abs(V0 - ref["solutions"])) <= 1e-9 * np.max(np.abs(ref["solutions"]))


def _cg_single(O, X, T, raw, tol, max_epochs):
    """Unpreconditioned CG of the worker above on one process."""
    n = X.shape[0]
    rows = np.arange(n, dtype=np.int32)

    def apply(v):
        return O.apply_rows(X, raw, rows, np.asfortranarray(v.astype(np.float32).astype(np.float64)))

    scales = np.sqrt((T ** 2).sum(0)) + 1e-12
    V = np.zeros_like(T)
    R = T - apply(V)
    d = R.copy()
    gamma = (R * R).sum(0)
    t = 0
    while t < max_epochs:
        ss = (R ** 2).sum(0)
        if np.sqrt(ss[0]) / scales[0] <= tol and np.mean(np.sqrt(ss[1:]) / scales[1:]) <= tol:
            break
        hd = apply(d)
        alpha = gamma / (d * hd).sum(0)
        V = V + d * alpha
        R = R - hd * alpha
        gnext = (R * R).sum(0)
        beta = np.where(gamma != 0.0, gnext / np.where(gamma != 0.0, gamma, 1.0), 0.0)
        gamma = gnext
        d = R + d * beta
        t += 1
    return t, V


def test_shard_partition_matches_library():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2405_18457_b200 import parallel as P
    for n, w in [(4096, 2), (43008, 2), (1835008, 8), (393216, 4), (100, 3)]:
        covered = []
        for r in range(w):
            a, b = P.shard_rows(n, w, r)
            assert (a, b) == P.shard_rows_c(n, w, r)
            assert a % 32 == 0 or a == n  # tiny n can leave trailing ranks empty (rejected by the optimiser)
            covered += list(range(a, b)) if n < 5000 else []
        if n < 5000:
            assert covered == list(range(n))
    for n in (1, 63, 64, 65, 300, 4096):
        T = (n + 63) // 64
        seen = sorted(P.tile_coords(L, n) for L in range(T * (T + 1) // 2))
        assert seen == sorted((a, b) for a in range(T) for b in range(a, T))


def test_world2_gloo_sharded_cg_and_gradient_match_single_process(oracle):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, t0, V0, F0, sh0), (_, t1, V1, F1, sh1) = res
    assert t0 == t1 and np.array_equal(V0, V1) and np.array_equal(F0, F1)  # identical decisions on both ranks
    assert sh0 == (0, 128) and sh1 == (128, 200)

    X, T, Z = _problem()
    raw = oracle.raw_from_constrained([0.9, 1.1, 1.3, 1.0, 0.5])
    # the same algorithm on one process (FP32 direction, serial column sums):
    # the decomposition changes only the order of the partial sums
    t_ref, V_ref = _cg_single(oracle, X, T, raw, 1e-4, 200)
    assert abs(t_ref - t0) <= 1
    if t_ref == t0:
        assert np.max(np.abs(V0 - V_ref)) <= 1e-5 * np.max(np.abs(V_ref))  # FP32 direction: order-level drift ~3e-7
    direct = np.linalg.solve(oracle.dense(X, raw), T)
    assert np.max(np.abs(V0 - direct)) <= 1e-2 * np.max(np.abs(direct))
    _, fz = oracle.quad_forms(X, raw, Z[:, :1], Z[:, :1], Z, Z)
    assert np.max(np.abs(F0 - fz) / np.abs(fz)) <= 1e-10
