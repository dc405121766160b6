"""The batched split of SURVEY.md §8e / BASELINE configs[4] ("config 2's batch sharded"):
P ranks each invert a contiguous shard [r B/P, (r+1) B/P) of the one seed-1 C2 batch with
no data-path collective, exactly as bench.py runs it.  Two processes share cuda:0 (gloo
for the gather only); every item's inverse, log|det| and sign must be BITWISE the
single-process result (items are independent: the row-parallel structure of Eq. (15),
PAPER.md L65-L67, puts nothing of one item into another)."""
import os
import socket
import tempfile

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

B = 12289          # ragged: not a multiple of the warp task or of P
SEED = 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard(total, world, rank):
    return total * rank // world, total * (rank + 1) // world


def _worker(rank, P, port, outdir):
    import torch
    import torch.distributed as tdist
    import paper_1401_7962_b200 as gj
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=P, init_method=f"tcp://127.0.0.1:{port}")
    try:
        lo, hi = _shard(B, P, rank)
        A = torch.from_numpy(synth.gen_c2_shard(lo, hi, seed=SEED)).cuda()
        r = gj.invert_batched(A, tol=32 * 2.0 ** -23)
        torch.cuda.synchronize()
        np.savez(os.path.join(outdir, f"r{rank}.npz"), lo=lo, hi=hi, inv=r.inverse.cpu().numpy(),
                 lg=r.logabsdet.cpu().numpy(), sign=r.sign.cpu().numpy(), info=r.info.cpu().numpy())
        tdist.barrier()
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_batch_bitwise_equals_one_process(P):
    import torch
    import torch.multiprocessing as mp
    import paper_1401_7962_b200 as gj
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(P, _free_port(), d), nprocs=P, join=True, start_method="spawn")
        parts = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(P)]
    A = torch.from_numpy(synth.gen_c2(batch=B, seed=SEED)).cuda()
    r1 = gj.invert_batched(A, tol=32 * 2.0 ** -23)
    torch.cuda.synchronize()
    inv1 = r1.inverse.cpu().numpy()
    lg1, sg1, in1 = r1.logabsdet.cpu().numpy(), r1.sign.cpu().numpy(), r1.info.cpu().numpy()
    covered = 0
    for p in parts:
        lo, hi = int(p["lo"]), int(p["hi"])
        covered += hi - lo
        assert np.array_equal(p["inv"].view(np.int32), inv1[lo:hi].view(np.int32)), (lo, hi)
        assert np.array_equal(p["lg"].view(np.int64), lg1[lo:hi].view(np.int64))
        assert np.array_equal(p["sign"], sg1[lo:hi])
        assert np.array_equal(p["info"], in1[lo:hi])
    assert covered == B
