"""GPU parity of the distributed large-n path (gj_dist_* through paper_1401_7962_b200/dist.py)
on the one GPU available: world size 1 (the full path, its all-to-all degenerate) and world
size 2 as two processes sharing cuda:0 over a gloo group (host-staged collectives, so the
two ranks' kernels never wait on one another).  Against the oracle, the exact Hadamard pin
and the single-GPU gj_invert (invariant P4)."""
import os
import socket
import tempfile

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, P, n, kind, port, outdir):
    import torch
    import torch.distributed as tdist
    from paper_1401_7962_b200.dist import invert_dist, local_columns
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=P, init_method=f"tcp://127.0.0.1:{port}")
    try:
        if kind == "gauss":
            A = synth.gen_gaussian(n, seed=70 + n)
        elif kind == "c5gen":
            A = synth.gen_gaussian(n, seed=4)      # the C5 generator (N(0,1)/sqrt(n), seed 4)
        else:
            A = synth.hadamard_pd(n, seed=5)[0]
        cols = local_columns(n, P, rank)
        A_local = torch.from_numpy(np.ascontiguousarray(A[:, cols])).cuda()
        r = invert_dist(A_local, n)
        torch.cuda.synchronize()
        np.savez(os.path.join(outdir, f"r{rank}.npz"), inv=r.inverse_local.cpu().numpy(), cols=np.array(cols),
                 lg=r.logabsdet, sign=r.sign, info=r.info, ipiv=r.ipiv.cpu().numpy())
    finally:
        tdist.destroy_process_group()


def run_dist(P, n, kind="gauss"):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(P, n, kind, _free_port(), d), nprocs=P, join=True, start_method="spawn")
        X = np.zeros((n, n))
        outs = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(P)]
        for o in outs:
            if len(o["cols"]):
                X[:, o["cols"]] = o["inv"]
        o0 = outs[0]
        return X, float(o0["lg"]), int(o0["sign"]), int(o0["info"]), o0["ipiv"]


def single(n, A):
    import torch
    import paper_1401_7962_b200 as gj
    r = gj.invert(torch.from_numpy(A).cuda(), tol=n * 2.0 ** -52)
    torch.cuda.synchronize()
    return r.inverse.cpu().numpy(), float(r.logabsdet), int(r.sign), r.ipiv.cpu().numpy()


@pytest.mark.parametrize("P,n", [(1, 300), (2, 300), (2, 1000), (1, 2048)])
def test_dist_gaussian(P, n):
    X, lg, sg, info, ipiv = run_dist(P, n)
    A = synth.gen_gaussian(n, seed=70 + n)
    ref = oracle.invert(A, tol=n * 2.0 ** -52)
    kappa = oracle.kappa_inf(A, ref.inverse[0])[0]
    e = np.abs(X - ref.inverse[0]).max() / np.abs(ref.inverse[0]).max()
    assert info == 0
    assert e <= max(1e-10, kappa * 2.0 ** -52), (e, kappa)
    assert np.array_equal(ipiv, ref.ipiv[0])
    assert sg == ref.sign[0]
    assert abs(lg - ref.logabsdet[0]) <= max(1e-10, kappa * 2.0 ** -52)
    # SURVEY §8e determinism target (invariant P4): the P-rank inverse is BITWISE the 1-GPU
    # one — every element sees the same panels, pivots and K-loop order whatever rank owns it
    Xs, lgs, sgs, ipivs = single(n, A)
    assert np.array_equal(ipiv, ipivs) and sg == sgs and lg == lgs
    assert np.array_equal(X, Xs)


@pytest.mark.parametrize("P", [1, 2])
def test_dist_hadamard_exact(P):
    n = 1024
    X, lg, sg, info, ipiv = run_dist(P, n, kind="hadamard")
    A = synth.hadamard_pd(n, seed=5)[0]
    assert np.array_equal(X, A.T / n)
    assert abs(lg - (n / 2) * np.log(n)) <= 1e-9


@pytest.mark.parametrize("P", [1, 2])
def test_dist_c5_generator_n8192_vs_stored_oracle(P):
    """oracle parity of the distributed code at n = 8192 on the C5 generator
    (seed 4): ipiv (R3), log|det| and sign (R4/R5), 64 sampled rows of the inverse (R1 kappa
    rule) and their residual (R2), against tests/golden/c4_oracle_ref_n8192_s4.npz (written by
    tools/make_c4_reference.py 8192 4: the long-double oracle, 1,174 s on 8 cores)."""
    from tests.parity import TOL_RES, ipiv_match
    ref = np.load(os.path.join(os.path.dirname(__file__), "golden", "c4_oracle_ref_n8192_s4.npz"))
    n = int(ref["n"])
    assert n == 8192 and int(ref["seed"]) == 4
    X, lg, sg, info, ipiv = run_dist(P, n, kind="c5gen")
    assert info == 0
    ok, _ = ipiv_match(ipiv, ref["ipiv"], ref["gap"])
    assert ok
    kappa = float(ref["kappa_inf"])
    rows = ref["rows"]
    e = np.abs(X[rows] - ref["inv_rows"]).max() / np.abs(ref["inv_rows"]).max()
    print(f"dist P={P} n=8192 seed 4: sampled-row rel err {e:.3e}, kappa_inf {kappa:.3e}")
    assert e <= max(1e-10, kappa * 2.0 ** -52)
    assert sg == int(ref["sign"])
    assert abs(lg - float(ref["logabsdet"])) <= max(1e-10, kappa * 2.0 ** -52)
    A = synth.gen_gaussian(n, seed=4)
    assert oracle.residual(A, X, rows=rows) <= TOL_RES[np.float64]


def _lib_worker(rank, P, n, kind, port, outdir):
    """The library-driven path (gj_dist_init / gj_invert_dist / gj_dist_finalize): the
    communicator and every collective inside libgjinv.so (NCCL)."""
    import torch
    import torch.distributed as tdist
    from paper_1401_7962_b200.dist import DistContext, local_columns
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=P, init_method=f"tcp://127.0.0.1:{port}")
    try:
        A = synth.gen_gaussian(n, seed=70 + n) if kind == "gauss" else synth.hadamard_pd(n, seed=5)[0]
        cols = local_columns(n, P, rank)
        A_local = torch.from_numpy(np.ascontiguousarray(A[:, cols])).cuda()
        with DistContext() as ctx:
            r = ctx.invert(A_local, n)
            r2 = ctx.invert(A_local, n)          # the handle is reusable
        torch.cuda.synchronize()
        assert torch.equal(r.inverse_local, r2.inverse_local)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), inv=r.inverse_local.cpu().numpy(), cols=np.array(cols),
                 lg=r.logabsdet, sign=r.sign, info=r.info, ipiv=r.ipiv.cpu().numpy())
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("n,kind", [(300, "gauss"), (1000, "gauss"), (1024, "hadamard")])
def test_library_driven_dist_one_rank(n, kind):
    """gj_invert_dist at P = 1 (one GPU): bitwise the single-GPU gj_invert (same panels, pivots
    and K-loop order) and exact on the Hadamard pin."""
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_lib_worker, args=(1, n, kind, _free_port(), d), nprocs=1, join=True, start_method="spawn")
        o = np.load(os.path.join(d, "r0.npz"))
    X = o["inv"]
    A = synth.gen_gaussian(n, seed=70 + n) if kind == "gauss" else synth.hadamard_pd(n, seed=5)[0]
    Xs, lgs, sgs, ipivs = single(n, A)
    assert int(o["info"]) == 0
    assert np.array_equal(X, Xs)
    assert np.array_equal(o["ipiv"], ipivs) and int(o["sign"]) == sgs and float(o["lg"]) == lgs
    if kind == "hadamard":
        assert np.array_equal(X, A.T / n)
