"""Exact rational brute-force oracles — TEST INFRASTRUCTURE ONLY.

These are the plain definitions of the two results Gauss–Jordan reaches exactly
(§2 III, Eqs. (12)–(13), L48–L54): the determinant by Laplace cofactor
expansion along the first row and the inverse as adjugate / determinant, in Python
``fractions.Fraction`` (`cofactor_det`, `adjugate_inverse`).
Factorial cost: intended for n ≤ 6 (the SPEC.md L420 sweep).  They share nothing with
the long-double Gauss–Jordan in ``gj_oracle.c``, which is why they can pin it.
"""
from __future__ import annotations

from fractions import Fraction
from typing import List, Sequence

Matrix = List[List[Fraction]]


def to_fractions(A: Sequence[Sequence]) -> Matrix:
    """Exact conversion (floats convert exactly via Fraction(float))."""
    return [[Fraction(x) if not isinstance(x, Fraction) else x for x in row] for row in A]


def _minor(A: Matrix, i: int, j: int) -> Matrix:
    return [row[:j] + row[j + 1:] for r, row in enumerate(A) if r != i]


def cofactor_det(A: Sequence[Sequence]) -> Fraction:
    """det A by Laplace expansion along the first row."""
    M = to_fractions(A)
    n = len(M)
    if n > 10:
        raise ValueError("cofactor_det: n > 10 (factorial cost guard, SPEC.md L283)")
    return _det(M)


def _det(M: Matrix) -> Fraction:
    n = len(M)
    if n == 0:
        return Fraction(1)
    if n == 1:
        return M[0][0]
    if n == 2:
        return M[0][0] * M[1][1] - M[0][1] * M[1][0]
    total = Fraction(0)
    for j in range(n):
        if M[0][j] == 0:
            continue
        c = M[0][j] * _det(_minor(M, 0, j))
        total += c if j % 2 == 0 else -c
    return total


def adjugate_inverse(A: Sequence[Sequence]) -> Matrix:
    """A⁻¹ = adj(A) / det A, adj(A)_ij = (−1)^{i+j} det(minor_ji).
    Raises ZeroDivisionError for an exactly singular A."""
    M = to_fractions(A)
    n = len(M)
    if n > 8:
        raise ValueError("adjugate_inverse: n > 8 (SPEC.md L293)")
    d = _det(M)
    if d == 0:
        raise ZeroDivisionError("singular: det = 0")
    inv = [[Fraction(0)] * n for _ in range(n)]
    for i in range(n):
        for j in range(n):
            c = _det(_minor(M, j, i))
            inv[i][j] = (c if (i + j) % 2 == 0 else -c) / d
    return inv


def permutation_sign(perm: Sequence[int]) -> int:
    """Sign of a permutation (0-based), by counting inversions — the textbook definition."""
    s = 1
    p = list(perm)
    for i in range(len(p)):
        for j in range(i + 1, len(p)):
            if p[i] > p[j]:
                s = -s
    return s
