"""Multi-GPU decomposition, exercised on CPU with gloo (world_size 2 and 3).

The sharded sweep (csrc/shard.cu) alternates node-row strips
(K(u), residual, RHS, time DFTs: all N slices local) and frequency blocks
(the block solves, full grid), with one halo exchange, one all-to-all each
way and rank-ordered scalar sums per sweep.  Here every rank takes its part
of the partition from the library's own planner (tp_shard_plan_make, a pure
host function), performs exactly those exchanges with torch.distributed
(gloo, CPU tensors) and uses the numpy oracle for the local arithmetic; the
gathered result must equal the single-process oracle sweep.
"""
import os
import socket
import sys

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def plan_of(cells, steps, P, r):
    from paper_2502_21013_b200 import shard_plan
    p = shard_plan(cells, steps, P, r)
    return dict(row0=p.row0, row1=p.row1, freq0=p.freq0, freq1=p.freq1, slice0=p.slice0,
                slice1=p.slice1, n_local=p.n_local)


@pytest.mark.parametrize("cells,steps", [(16, 8), (32, 12), (256, 256), (2048, 1024)])
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_partition_covers_everything_once(cells, steps, P):
    m, K = cells - 1, steps // 2 + 1
    if K < P or m < P:
        with pytest.raises(ValueError, match="more ranks"):
            plan_of(cells, steps, P, 0)
        return
    plans = [plan_of(cells, steps, P, r) for r in range(P)]
    assert plans[0]["row0"] == 0 and plans[-1]["row1"] == m
    assert plans[0]["freq0"] == 0 and plans[-1]["freq1"] == K
    assert plans[0]["slice0"] == 0 and plans[-1]["slice1"] == steps
    for a, b in zip(plans, plans[1:]):
        assert a["row1"] == b["row0"] and a["freq1"] == b["freq0"] and a["slice1"] == b["slice0"]
    for p in plans:
        assert p["row1"] > p["row0"] and p["freq1"] > p["freq0"] and p["slice1"] > p["slice0"]
        assert p["n_local"] == (p["row1"] - p["row0"]) * m


@pytest.mark.parametrize("steps,P", [(1024, 8), (1024, 2), (256, 4), (63, 3)])
def test_frequency_order_is_a_balanced_permutation(steps, P):
    """Snake-dealt frequencies: a permutation of 0..N/2, each
    rank's slots contiguous, every rank a spread of the spectrum (its mean
    frequency within one round of the global mean) and a balanced share of
    odd harmonics (the only ones that iterate under odd-symmetric sources)."""
    from paper_2502_21013_b200 import shard_freq_order
    K = steps // 2 + 1
    order = shard_freq_order(2049, steps, P)
    assert sorted(order.tolist()) == list(range(K))
    plans = [plan_of(2049, steps, P, r) for r in range(P)]
    odd = []
    for p in plans:
        ks = order[p["freq0"]:p["freq1"]]
        assert abs(ks.mean() - (K - 1) / 2) <= P
        odd.append(int(np.sum(ks % 2)))
    assert max(odd) - min(odd) <= 2
    assert np.array_equal(shard_freq_order(2049, steps, 1), np.arange(K))


def test_partition_rejects_too_many_ranks():
    from paper_2502_21013_b200 import shard_plan
    with pytest.raises(ValueError):
        shard_plan(4, 8, 5, 0)  # 3 grid rows for 5 ranks


# ---------------------------------------------------------------- emulation

def _worker(rank, world, port, cells, steps, out_path):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import tp_oracle as O
    from paper_2502_21013_b200 import baseline_desc

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    d = baseline_desc(0)
    d.cells, d.steps = cells, steps
    g = O.GridSetup(d)
    m, n, N = g.m, g.n, g.N
    K = N // 2 + 1
    plans = [plan_of(cells, steps, world, r) for r in range(world)]
    me = plans[rank]
    rows = slice(me["row0"] * m, me["row1"] * m)
    rng = np.random.default_rng(0)
    U_full = rng.standard_normal((N, n)) * 0.05
    F = g.loads()
    nu_hat = np.array([3.0, 2.0, 5.0, 1.0, 1.0])
    Kh = g.stiffness_frozen(nu_hat)
    mass = g.mass_diag()
    U = U_full[:, rows].copy()  # my strip, all N slices

    def sendrecv(send, peer, shape):
        out = torch.empty(shape, dtype=torch.float64)
        reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(send)), peer),
                dist.irecv(out, peer)]
        for r_ in reqs:
            r_.wait()
        return out.numpy()

    # 1. halo rows (N x m each side), zero at the outer boundary
    lo = np.zeros((N, m))
    hi = np.zeros((N, m))
    ops = []
    if rank > 0:
        lo = sendrecv(U[:, :m], rank - 1, (N, m))
    if rank < world - 1:
        hi = sendrecv(U[:, -m:], rank + 1, (N, m))
    # 2. K(u) / residual / RHS on my strip: embed strip + halo in a zero field
    emb = np.zeros((N, n))
    emb[:, rows] = U
    if rank > 0:
        emb[:, (me["row0"] - 1) * m:me["row0"] * m] = lo
    if rank < world - 1:
        emb[:, me["row1"] * m:(me["row1"] + 1) * m] = hi
    KU = g.apply_k(emb)[:, rows]
    KhU = (Kh @ emb.T).T[:, rows]
    Floc = F[:, rows]
    G = Floc + KhU - KU
    R = Floc - mass[rows] * ((U - np.roll(U, 1, axis=0)) / g.tau) - KU
    r2 = torch.tensor([float(np.sum(R * R))], dtype=torch.float64)
    parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, r2)
    res_norm = float(np.sqrt(sum(float(p.item()) for p in parts)))  # rank order
    # 3. forward DFT along time (local), half spectrum K x n_r, stored in the
    # library's slot order (snake-dealt frequencies, tp_shard_freq_order)
    from paper_2502_21013_b200 import shard_freq_order
    order = shard_freq_order(cells, steps, world)
    Gh = np.fft.fft(G, axis=0)[:K][order]
    # 4. all-to-all strips -> frequency blocks
    Ghf = np.zeros((me["freq1"] - me["freq0"], n), dtype=complex)
    for q in range(world):
        pq = plans[q]
        blk = Gh[pq["freq0"]:pq["freq1"]]
        if q == rank:
            got = blk
        else:
            sh = (me["freq1"] - me["freq0"], (pq["row1"] - pq["row0"]) * m, 2)
            got = sendrecv(np.stack([blk.real, blk.imag], -1), q, sh)
            got = got[..., 0] + 1j * got[..., 1]
        Ghf[:, pq["row0"] * m:pq["row1"] * m] = got
    # 5. solve my frequencies on the full grid
    Uhf = np.zeros_like(Ghf)
    for kk, slot in enumerate(range(me["freq0"], me["freq1"])):
        lam = O.symbol(int(order[slot]), N, g.tau)
        A = (lam * sp.diags(mass) + Kh).astype(complex).tocsc()
        Uhf[kk] = spla.spsolve(A, Ghf[kk])
    # 6. all-to-all back, inverse DFT of my strip
    Uh = np.zeros((K, me["n_local"]), dtype=complex)
    for q in range(world):
        pq = plans[q]
        blk = Uhf[:, pq["row0"] * m:pq["row1"] * m]
        if q == rank:
            got = blk
        else:
            sh = (pq["freq1"] - pq["freq0"], me["n_local"], 2)
            got = sendrecv(np.stack([blk.real, blk.imag], -1), q, sh)
            got = got[..., 0] + 1j * got[..., 1]
        Uh[pq["freq0"]:pq["freq1"]] = got
    Uh = Uh[np.argsort(order)]  # slot order -> frequency order
    full = np.zeros((N, me["n_local"]), dtype=complex)
    full[:K] = Uh
    for k in range(1, (N + 1) // 2):
        full[N - k] = np.conj(Uh[k])
    Unew = np.fft.ifft(full, axis=0).real
    # 7. gather strips on rank 0
    out = [torch.zeros((N, plans[q]["n_local"]), dtype=torch.float64) for q in range(world)]
    if rank == 0:
        for q in range(1, world):
            dist.recv(out[q], q)
        out[0] = torch.from_numpy(Unew)
        np.savez(out_path, U=np.concatenate([o.numpy() for o in out], axis=1), res=res_norm)
    else:
        dist.send(torch.from_numpy(np.ascontiguousarray(Unew)), 0)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sweep_matches_single_process(tmp_path, world):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    from oracle import tp_oracle as O
    from paper_2502_21013_b200 import baseline_desc

    cells, steps = 16, 8
    out = str(tmp_path / "u.npz")
    mp.spawn(_worker, args=(world, free_port(), cells, steps, out), nprocs=world, join=True)
    got = np.load(out)
    # single-process oracle: the same sweep on the full field
    d = baseline_desc(0)
    d.cells, d.steps = cells, steps
    g = O.GridSetup(d)
    U0 = np.random.default_rng(0).standard_normal((g.N, g.n)) * 0.05
    F = g.loads()
    Kh = g.stiffness_frozen(np.array([3.0, 2.0, 5.0, 1.0, 1.0]))
    res = O.block_l2(O.residual(g, U0, F))
    G = F + (Kh @ U0.T).T - g.apply_k(U0)
    U1 = O.PeriodicSolver(sp.diags(g.mass_diag()), Kh, g.tau, g.N).solve(G)
    assert abs(float(got["res"]) - res) <= 1e-13 * res
    assert np.linalg.norm(got["U"] - U1) <= 1e-12 * np.linalg.norm(U1)
