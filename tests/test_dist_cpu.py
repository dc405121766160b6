"""Host logic of the distributed large-n path (paper_1401_7962_b200/dist.py) on CPU:
world-size 1, 2 and 3 ``gloo`` process groups over 127.0.0.1, the compute steps supplied
by tests/dist_steps_ref.py.  Checks the block-cyclic layout, the per-panel broadcasts and
the un-permutation all-to-all against the oracle (P4: 1 rank == P ranks)."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1401_7962_b200.dist import BLOCK, invert_dist, local_columns, owner


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, P, n, kind, port, outdir):
    from tests.dist_steps_ref import RefSteps
    tdist.init_process_group("gloo", rank=rank, world_size=P, init_method=f"tcp://127.0.0.1:{port}")
    try:
        A = synth.gen_gaussian(n, seed=60 + n) if kind == "gauss" else synth.hadamard_pd(n, seed=5)[0]
        cols = local_columns(n, P, rank)
        A_local = torch.from_numpy(np.ascontiguousarray(A[:, cols]))
        r = invert_dist(A_local, n, steps=RefSteps(n, P, rank))
        np.savez(os.path.join(outdir, f"r{rank}.npz"), inv=r.inverse_local.numpy(), cols=np.array(cols),
                 lg=r.logabsdet, sign=r.sign, info=r.info, ipiv=r.ipiv.numpy())
    finally:
        tdist.destroy_process_group()


def run_dist(P, n, kind="gauss"):
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(P, n, kind, _free_port(), d), nprocs=P, join=True, start_method="spawn")
        X = np.zeros((n, n))
        outs = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(P)]
        for o in outs:
            if len(o["cols"]):
                X[:, o["cols"]] = o["inv"]
        o0 = outs[0]
        for o in outs[1:]:   # replicated outputs agree on every rank
            assert float(o["lg"]) == float(o0["lg"]) and int(o["sign"]) == int(o0["sign"])
            assert np.array_equal(o["ipiv"], o0["ipiv"])
        return X, float(o0["lg"]), int(o0["sign"]), int(o0["info"]), o0["ipiv"]


def test_block_cyclic_layout():
    n, P = 1000, 3
    cols = [local_columns(n, P, r) for r in range(P)]
    assert sorted(c for cs in cols for c in cs) == list(range(n))
    for r in range(P):
        assert all(owner(c, P) == r for c in cols[r])
        assert all((c // BLOCK) % P == r for c in cols[r])


@pytest.mark.parametrize("P", [1, 2, 3])
def test_gaussian_matches_oracle(P):
    n = 300    # npad 384: three panels, ragged real tail
    X, lg, sg, info, ipiv = run_dist(P, n)
    A = synth.gen_gaussian(n, seed=60 + n)
    ref = oracle.invert(A, tol=n * 2.0 ** -52)
    kappa = oracle.kappa_inf(A, ref.inverse[0])[0]
    e = np.abs(X - ref.inverse[0]).max() / np.abs(ref.inverse[0]).max()
    assert info == 0
    assert e <= max(1e-10, kappa * 2.0 ** -52), (e, kappa)
    assert np.array_equal(ipiv, ref.ipiv[0])
    assert sg == ref.sign[0]
    assert abs(lg - ref.logabsdet[0]) <= 1e-10


def test_hadamard_exact_two_ranks():
    """P6 through the distributed host logic: every step an exact tie, inverse A^T / n."""
    n = 256
    X, lg, sg, info, ipiv = run_dist(2, n, kind="hadamard")
    A = synth.hadamard_pd(n, seed=5)[0]
    assert np.array_equal(X, A.T / n)
    assert abs(lg - (n / 2) * np.log(n)) <= 1e-9
