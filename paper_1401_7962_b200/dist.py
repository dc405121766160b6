"""Distributed large-n Gauss–Jordan inversion: one matrix, column-block-cyclic over the
ranks of a ``torch.distributed`` process group (BASELINE.json configs[4]).

Plumbing only.  Every compute step is a C-ABI call of ``libgjinv.so`` (``include/gjinv.h``,
``gj_dist_*``); this module allocates the per-rank buffers and moves them between ranks
with ``torch.distributed`` (NCCL over NVLink on a GPU box):

* global column block j (``BLOCK`` = 128 columns, the panel width) lives on rank j % P;
  rows are complete on every rank, so a panel's max-|a_ik| pivot search (PAPER.md Obs. 3,
  L60) is local to the panel's owner;
* per panel k: the owner factors it (``gj_dist_step_factor``: the panel's 128 pivot steps,
  Eqs. (14)-(15) restricted to the panel), then ONE broadcast of W (the factored panel)
  and the replicated step record / row positions goes from the owner to every rank, and
  every rank applies the panel's aggregated rank-128 update to its own columns
  (``gj_dist_step_update``: DMMA GEMM);
* the listing's un-permutation (L179-L198) is one all-to-all of columns at the end.

The step functions are reached through a ``steps`` object so that the host logic can be
exercised on CPU with world-size-2 ``gloo`` tests (``tests/test_dist_cpu.py`` supplies a
CPU stand-in for the steps there; the product path only ever uses :class:`CudaSteps`,
which fails loudly without the CUDA library).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional

import torch
import torch.distributed as tdist

BLOCK = 128
MAX_RANKS = 8


def owner(gc: int, P: int) -> int:
    return (gc // BLOCK) % P


def local_columns(n: int, P: int, rank: int) -> List[int]:
    """Global real columns (< n) held by ``rank``, in increasing order (the layout of
    ``A_local`` and of the returned inverse)."""
    return [c for c in range(n) if owner(c, P) == rank]


def sizes(n: int, P: int, rank: int):
    """(npad, padded local columns, real local columns)."""
    npad = (n + BLOCK - 1) // BLOCK * BLOCK
    nb = npad // BLOCK
    nl = ((nb - rank + P - 1) // P) * BLOCK
    return npad, nl, len(local_columns(n, P, rank))


class CudaSteps:
    """The distributed steps through the C-ABI (device tensors, current stream)."""

    def __init__(self, n: int, P: int, rank: int):
        from . import lib, _check
        self.lib, self._check = lib, _check
        self.n, self.P, self.rank = n, P, rank
        for name, args in (
            ("gj_dist_sizes", [ctypes.c_int] * 3 + [ctypes.c_void_p] * 3),
            ("gj_dist_step_init", [ctypes.c_int] * 3 + [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 5),
            ("gj_dist_step_factor", [ctypes.c_int] * 4 + [ctypes.c_void_p] * 8),
            ("gj_dist_step_update", [ctypes.c_int] * 5 + [ctypes.c_void_p] * 6),
            ("gj_dist_step_finalize", [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double] + [ctypes.c_void_p] * 6),
            ("gj_dist_step_unpermute_plan", [ctypes.c_int] * 3 + [ctypes.c_void_p] * 5),
            ("gj_dist_step_unpermute_pack", [ctypes.c_int] * 3 + [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
            ("gj_dist_step_unpermute_unpack", [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_int64, ctypes.c_void_p]),
        ):
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ctypes.c_int

    @staticmethod
    def _p(t):
        return None if t is None else t.data_ptr()

    def _s(self):
        return torch.cuda.current_stream().cuda_stream

    def init(self, A_local, lda, X, pos, pivstep, smax):
        self._check(self.lib.gj_dist_step_init(self.n, self.P, self.rank, self._p(A_local), lda, X.data_ptr(), pos.data_ptr(),
                                          pivstep.data_ptr(), smax.data_ptr(), self._s()))

    def factor(self, k, X, pos, pivstep, rec_p, rec_q, rec_row, W):
        self._check(self.lib.gj_dist_step_factor(self.n, self.P, self.rank, k, X.data_ptr(), pos.data_ptr(), pivstep.data_ptr(),
                                            rec_p.data_ptr(), rec_q.data_ptr(), rec_row.data_ptr(), W.data_ptr(), self._s()))

    def update(self, k, part, X, W, pivstep, rec_row, R):
        self._check(self.lib.gj_dist_step_update(self.n, self.P, self.rank, k, part, self._p(X), W.data_ptr(),
                                            pivstep.data_ptr(), rec_row.data_ptr(), self._p(R), self._s()))

    def finalize(self, rec_p, rec_q, tol, smax, ipiv, logabsdet, sign, info):
        self._check(self.lib.gj_dist_step_finalize(self.n, rec_p.data_ptr(), rec_q.data_ptr(), tol, smax.data_ptr(),
                                              ipiv.data_ptr(), logabsdet.data_ptr(), sign.data_ptr(), info.data_ptr(),
                                              self._s()))

    def plan(self, pivstep, send_cols, recv_cols, counts):
        self._check(self.lib.gj_dist_step_unpermute_plan(self.n, self.P, self.rank, pivstep.data_ptr(), send_cols.data_ptr(),
                                                    recv_cols.data_ptr(), counts.data_ptr(), self._s()))

    def pack(self, X, rec_row, send_cols, m, sendbuf):
        self._check(self.lib.gj_dist_step_unpermute_pack(self.n, self.P, self.rank, self._p(X), rec_row.data_ptr(),
                                                    send_cols.data_ptr(), m, self._p(sendbuf), self._s()))

    def unpack(self, recvbuf, recv_cols, m, Y, ld):
        self._check(self.lib.gj_dist_step_unpermute_unpack(self.n, self._p(recvbuf), recv_cols.data_ptr(), m, self._p(Y), ld,
                                                      self._s()))


@dataclass
class DistResult:
    inverse_local: torch.Tensor   # n x len(local_columns(n, P, rank)): this rank's columns of A^-1
    logabsdet: float
    sign: int
    info: int
    ipiv: torch.Tensor            # [n] int32, LAPACK-style 1-based (replicated)
    timings: dict


def _collective(group, device):
    """NCCL moves device tensors directly; other backends (gloo) stage through host memory."""
    backend = tdist.get_backend(group)
    staged = backend != "nccl" and device.type == "cuda"

    def bcast(t, src):
        if staged:
            h = t.cpu()
            tdist.broadcast(h, src=tdist.get_global_rank(group, src) if group is not None else src, group=group)
            t.copy_(h)
        else:
            tdist.broadcast(t, src=tdist.get_global_rank(group, src) if group is not None else src, group=group)

    def allreduce_max(t):
        if staged:
            h = t.cpu()
            tdist.all_reduce(h, op=tdist.ReduceOp.MAX, group=group)
            t.copy_(h)
        else:
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX, group=group)

    def all_to_all(out, inp, out_splits, in_splits):
        if staged:
            ho = torch.empty(out.shape, dtype=out.dtype)
            tdist.all_to_all_single(ho, inp.cpu(), out_splits, in_splits, group=group)
            out.copy_(ho)
        else:
            tdist.all_to_all_single(out, inp, out_splits, in_splits, group=group)

    return bcast, allreduce_max, all_to_all


def invert_dist(A_local: torch.Tensor, n: int, *, group=None, tol: Optional[float] = None, steps=None,
                timing: bool = False) -> DistResult:
    """Invert the n x n fp64 matrix whose block-cyclic columns ``local_columns(n, P, rank)``
    this rank holds in ``A_local`` (n x ncols, row-major; CUDA for the product path).
    Collective over ``group`` (default: the world).  Returns this rank's columns of A^-1."""
    P = tdist.get_world_size(group)
    rank = tdist.get_rank(group)
    if P > MAX_RANKS:
        raise ValueError(f"at most {MAX_RANKS} ranks")
    if n <= 64:
        raise ValueError("the distributed path is for n > 64 (use invert_batched)")
    device = A_local.device
    if steps is None:
        if device.type != "cuda":
            raise ValueError("A_local must be a CUDA tensor (there is no CPU fallback)")
        steps = CudaSteps(n, P, rank)
    npad, nl, nr = sizes(n, P, rank)
    if A_local.dtype != torch.float64 or A_local.shape != (n, nr) or (nr and A_local.stride(1) != 1):
        raise ValueError(f"A_local must be float64 [{n}, {nr}] with unit column stride")
    bcast, allreduce_max, all_to_all = _collective(group, device)
    f64 = dict(dtype=torch.float64, device=device)
    i32 = dict(dtype=torch.int32, device=device)
    X = torch.empty((npad, max(nl, 1)), **f64)
    # replicated state, broadcast by the panel owner as one int32 buffer:
    # pos | pivstep | rec_q | rec_row | rec_p (fp64 viewed as 2 x int32).  Double-buffered by
    # panel parity like W: panel k+1's broadcast lands in the buffer panel k-1's update read,
    # never in the one panel k's update (running beside it) still reads.
    ibufs = [torch.empty(6 * npad, **i32) for _ in range(2)]

    def views(ib):
        return (ib[:npad], ib[npad:2 * npad], ib[2 * npad:3 * npad], ib[3 * npad:4 * npad],
                ib[4 * npad:].view(torch.float64))

    # the factored panel W, double-buffered: W_{k+1} arrives while panel k's update still reads W_k
    wbuf = [torch.empty((npad, BLOCK), **f64) for _ in range(2)]
    R = torch.empty((BLOCK, max(nl, 1)), **f64)
    smax = torch.zeros(1, dtype=torch.int64, device=device)
    ev = []
    cuda = device.type == "cuda"
    main = torch.cuda.current_stream(device) if cuda else None
    side = torch.cuda.Stream(device=device) if cuda else None

    def mark(name):
        if timing and cuda:
            e = torch.cuda.Event(enable_timing=True)
            e.record(main)
            ev.append((name, e))

    def record(stream):
        if not cuda:
            return None
        e = torch.cuda.Event()
        e.record(stream)
        return e

    mark("start")
    nb = npad // BLOCK
    pos, pivstep, rec_q, rec_row, rec_p = views(ibufs[0])
    steps.init(A_local if nr else None, max(nr, 1), X, pos, pivstep, smax)
    allreduce_max(smax)   # bit patterns of non-negative doubles order like the values
    Xo = X if nl else None
    Ro = R if nl else None
    # panel 0: factored and broadcast before the loop
    if rank == 0:
        steps.factor(0, X, pos, pivstep, rec_p, rec_q, rec_row, wbuf[0])
    if P > 1:
        bcast(ibufs[0], 0)
        bcast(wbuf[0], 0)
    ev_upd = record(main)
    for k in range(nb):
        W = wbuf[k % 2]
        _, pivstep, _, rec_row, _ = views(ibufs[k % 2])
        nxt = k + 1 < nb
        own_next = nxt and (k + 1) % P == rank
        ev_fac = None
        if own_next:
            # look-ahead: panel k+1's columns first, factor it (on a copy of the state in the
            # other buffer), then the rest of panel k's update runs beside that factorisation
            steps.update(k, 1, Xo, W, pivstep, rec_row, Ro)
            ibufs[(k + 1) % 2].copy_(ibufs[k % 2])
            npos, npiv, nrq, nrr, nrp = views(ibufs[(k + 1) % 2])
            steps.factor(k + 1, X, npos, npiv, nrp, nrq, nrr, wbuf[(k + 1) % 2])
            ev_fac = record(main)
            steps.update(k, 2, Xo, W, pivstep, rec_row, Ro)
        else:
            steps.update(k, 0, Xo, W, pivstep, rec_row, Ro)
        if nxt and P > 1:
            # panel k+1 travels on a side stream into the buffers of parity k+1: after its
            # factorisation (owner) and after panel k-1's update, their last reader — not after
            # panel k's update, which reads the other parity
            if cuda:
                side.wait_event(ev_upd)
                if ev_fac is not None:
                    side.wait_event(ev_fac)
                with torch.cuda.stream(side):
                    bcast(ibufs[(k + 1) % 2], (k + 1) % P)
                    bcast(wbuf[(k + 1) % 2], (k + 1) % P)
                ev_b = record(side)
                ev_upd = record(main)
                main.wait_event(ev_b)
            else:
                bcast(ibufs[(k + 1) % 2], (k + 1) % P)
                bcast(wbuf[(k + 1) % 2], (k + 1) % P)
        elif cuda:
            ev_upd = record(main)
    mark("eliminated")
    pos, pivstep, rec_q, rec_row, rec_p = views(ibufs[(nb - 1) % 2])
    ipiv = torch.empty(n, **i32)
    lg = torch.empty(1, **f64)
    sg = torch.empty(1, dtype=torch.int8, device=device)
    info = torch.empty(1, **i32)
    steps.finalize(rec_p, rec_q, -1.0 if tol is None else float(tol), smax, ipiv, lg, sg, info)
    # un-permutation: Ainv[i][j] = X[rec_row[i]][pivstep[j]], one all-to-all of columns
    send_cols = torch.empty(max(nl, 1), **i32)
    recv_cols = torch.empty(max(nr, 1), **i32)
    counts = torch.empty(2 * P, **i32)
    steps.plan(pivstep, send_cols, recv_cols, counts)
    cnt = counts.cpu().tolist()
    ms, mr = sum(cnt[:P]), sum(cnt[P:])
    sendbuf = torch.empty((max(ms, 1), n), **f64)
    recvbuf = torch.empty((max(mr, 1), n), **f64)
    steps.pack(X if ms else None, rec_row, send_cols, ms, sendbuf if ms else None)
    if P > 1:
        all_to_all(recvbuf[:mr], sendbuf[:ms], cnt[P:], cnt[:P])
    else:
        recvbuf = sendbuf
    Y = torch.empty((n, nr), **f64)
    steps.unpack(recvbuf if mr else None, recv_cols, mr, Y if nr else None, max(nr, 1))
    mark("done")
    times = {}
    if ev:
        torch.cuda.synchronize(device)
        t0 = ev[0][1]
        times = {name: t0.elapsed_time(e) for name, e in ev[1:]}
    return DistResult(Y, float(lg.item()), int(sg.item()), int(info.item()), ipiv, times)


class DistContext:
    """The library-driven NCCL path (``gj_dist_init`` / ``gj_invert_dist`` /
    ``gj_dist_finalize``): the same schedule as :func:`invert_dist`, with the communicator and
    the per-panel exchange inside ``libgjinv.so``.  Collective over ``group`` (default: the
    world); rank 0 creates the NCCL unique id and the group broadcasts it."""

    def __init__(self, group=None, device: Optional[torch.device] = None):
        from . import lib, _check
        self.lib, self._check = lib, _check
        self.P = tdist.get_world_size(group)
        self.rank = tdist.get_rank(group)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        uid = (ctypes.c_ubyte * 128)()
        if self.rank == 0:
            _check(lib.gj_dist_get_unique_id(uid))
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
        if tdist.get_backend(group) == "nccl":
            t = t.to(dev)
        tdist.broadcast(t, src=tdist.get_global_rank(group, 0) if group is not None else 0, group=group)
        buf = (ctypes.c_ubyte * 128)(*t.cpu().tolist())
        self.handle = ctypes.c_void_p()
        _check(lib.gj_dist_init(self.P, self.rank, buf, dev.index, ctypes.byref(self.handle)))

    def invert(self, A_local: torch.Tensor, n: int, tol: Optional[float] = None, stream=None) -> "DistResult":
        """This rank's columns of A^-1 (``local_columns(n, P, rank)``), fp64, on the context's device."""
        npad, nl, nr = sizes(n, self.P, self.rank)
        if A_local.dtype != torch.float64 or A_local.shape != (n, nr) or A_local.device != self.device or \
                (nr and A_local.stride(1) != 1):
            raise ValueError(f"A_local must be float64 [{n}, {nr}] on {self.device} with unit column stride")
        f64 = dict(dtype=torch.float64, device=self.device)
        Y = torch.empty((n, nr), **f64)
        ipiv = torch.empty(n, dtype=torch.int32, device=self.device)
        lg = torch.empty(1, **f64)
        sg = torch.empty(1, dtype=torch.int8, device=self.device)
        info = torch.empty(1, dtype=torch.int32, device=self.device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._check(self.lib.gj_invert_dist(self.handle, n, A_local.data_ptr() if nr else None, max(A_local.stride(0), 1),
                                            Y.data_ptr() if nr else None, max(nr, 1), ipiv.data_ptr(), lg.data_ptr(),
                                            sg.data_ptr(), info.data_ptr(), -1.0 if tol is None else float(tol),
                                            s.cuda_stream))
        return DistResult(Y, float(lg.item()), int(sg.item()), int(info.item()), ipiv, {})

    def close(self):
        if self.handle:
            self._check(self.lib.gj_dist_finalize(self.handle))
            self.handle = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
