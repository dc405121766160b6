"""CPU stand-in for the distributed steps (test infrastructure, tests/ only).

Implements, in plain torch CPU float64, the same step contract as ``gj_dist_*``
(include/gjinv.h) so that the host orchestration in ``paper_1401_7962_b200/dist.py``
(block-cyclic layout, broadcasts, the un-permutation all-to-all) can be run with
world-size-2 ``gloo`` process groups on a machine without a GPU.  It shares no code with
the CUDA path; each step restates the paper's method directly:

* factor: the textbook Gauss–Jordan step (§2 Eqs. (14)-(15), L61-L72) with the
  max-|a_ik| pivot among the un-pivoted rows (Obs. 3, L60), ties to the smallest position
  of the listing's swapped array (L151-L162, reading G3), restricted to the panel's
  columns (compact storage: column k becomes the D column);
* update: the panel's rank-128 aggregate X += W R - S R;
* finalize: Eq. (13) with the swap sign (G4); plan / pack / unpack: Ainv[i][j] =
  X[rec_row[i]][pivstep[j]] (the listing's un-permutation, L179-L198).
"""
from __future__ import annotations

import math

import torch

from paper_1401_7962_b200.dist import BLOCK, owner, sizes


def _gcol(lc, P, rank):
    return ((lc // BLOCK) * P + rank) * BLOCK + lc % BLOCK


def _lcol(gc, P):
    return (gc // BLOCK // P) * BLOCK + gc % BLOCK


class RefSteps:
    def __init__(self, n, P, rank):
        self.n, self.P, self.rank = n, P, rank
        self.npad, self.nl, self.nr = sizes(n, P, rank)

    def init(self, A_local, lda, X, pos, pivstep, smax):
        n, npad = self.n, self.npad
        X.zero_()
        m = 0.0
        for lc in range(self.nl):
            gc = _gcol(lc, self.P, self.rank)
            if gc < n:
                X[:n, lc] = A_local[:, lc]
                m = max(m, float(A_local[:, lc].abs().max()))
            else:
                X[gc, lc] = 1.0
        pos.copy_(torch.arange(npad, dtype=torch.int32))
        pivstep.fill_(-1)
        smax.copy_(torch.tensor([m], dtype=torch.float64).view(torch.int64))

    def factor(self, k, X, pos, pivstep, rec_p, rec_q, rec_row, W):
        c0 = (k // self.P) * BLOCK
        J = slice(c0, c0 + BLOCK)
        for s in range(BLOCK):
            kg = k * BLOCK + s
            col = X[:, c0 + s]
            elig = pivstep < 0
            a = torch.where(elig, col.abs(), torch.full_like(col, -1.0))
            mval = a.max()
            cand = torch.nonzero(a == mval).flatten()
            r = int(cand[torch.argmin(pos[cand])])
            p = float(X[r, c0 + s])
            q = int(pos[r])
            rec_p[kg], rec_q[kg], rec_row[kg] = p, q, r
            at_k = torch.nonzero(pos == kg).flatten()
            if len(at_k):
                pos[at_k[0]] = q
            pos[r] = kg
            pivstep[r] = kg
            f = X[:, c0 + s].clone()
            rowp = X[r, J] / p
            rowp[s] = 1.0 / p
            X[:, J] -= torch.outer(f, rowp)
            X[:, c0 + s] = -f / p
            X[r, J] = rowp
        W.copy_(X[:, J])

    def update(self, k, part, X, W, pivstep, rec_row, R):
        """part 0: all local columns but the own panel k; part 1: gather R, then only the
        local columns of panel k+1; part 2: the rest (R from part 1)."""
        if X is None:
            return
        k0 = k * BLOCK
        rows = rec_row[k0:k0 + BLOCK].long()
        if part != 2:
            R.copy_(X[rows, :])
        cols = torch.ones(self.nl, dtype=torch.bool)
        if k % self.P == self.rank:
            cols[(k // self.P) * BLOCK:(k // self.P + 1) * BLOCK] = False
        nxt = torch.zeros(self.nl, dtype=torch.bool)
        if part > 0:
            c1 = ((k + 1) // self.P) * BLOCK
            nxt[c1:c1 + BLOCK] = True
        if part == 1:
            cols = nxt
        elif part == 2:
            cols &= ~nxt
        idx = torch.nonzero(cols).flatten()
        upd = X[:, idx] + W @ R[:, idx]
        upd[rows] -= R[:, idx]
        X[:, idx] = upd

    def finalize(self, rec_p, rec_q, tol, smax, ipiv, logabsdet, sign, info):
        n = self.n
        s = float(smax.view(torch.float64)[0])
        tau = (n * 2.0 ** -52 if tol < 0 else tol) * s
        lg, par, first = 0.0, 0, 0
        for k in range(n):
            p, q = float(rec_p[k]), int(rec_q[k])
            ipiv[k] = q + 1
            lg += math.log(abs(p)) if p != 0 else -math.inf
            par ^= int(q != k) ^ int(p < 0)
            if first == 0 and abs(p) <= tau:
                first = k + 1
        info[0] = first
        logabsdet[0] = -math.inf if first else lg
        sign[0] = 0 if first else (-1 if par else 1)

    def plan(self, pivstep, send_cols, recv_cols, counts):
        n, P, rank = self.n, self.P, self.rank
        send = [[] for _ in range(P)]
        recv = [[] for _ in range(P)]
        for j in range(n):
            c = int(pivstep[j])
            src, dst = owner(c, P), owner(j, P)
            if src == rank:
                send[dst].append(_lcol(c, P))
            if dst == rank:
                recv[src].append(_lcol(j, P))
        sc = [c for d in send for c in d]
        rc = [c for d in recv for c in d]
        send_cols[:len(sc)] = torch.tensor(sc, dtype=torch.int32)
        recv_cols[:len(rc)] = torch.tensor(rc, dtype=torch.int32)
        counts.copy_(torch.tensor([len(d) for d in send] + [len(d) for d in recv], dtype=torch.int32))

    def pack(self, X, rec_row, send_cols, m, sendbuf):
        if m == 0:
            return
        rows = rec_row[:self.n].long()
        sendbuf[:m] = X[rows][:, send_cols[:m].long()].T

    def unpack(self, recvbuf, recv_cols, m, Y, ld):
        if m == 0:
            return
        Y[:, recv_cols[:m].long()] = recvbuf[:m].T
