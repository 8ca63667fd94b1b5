"""Oracle, part 1: the transform matrices, the fast factorisation and the
matrix-level figures of merit of arXiv 1606.05562.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy, float64 or
exact Python/numpy integers.  Each object cites the PAPER.md lines it restates.
"""
from __future__ import annotations

import math

import numpy as np

N = 16

# --------------------------------------------------------------------------
# §2, PAPER.md:270-287 — the proposed low-complexity matrix T, typed row by row
# exactly as printed.
# --------------------------------------------------------------------------
_T_ROWS = """
1 1 1 1 1 1 1 1 1 1 1 1 1 1 1 1
1 1 1 1 1 1 1 1 -1 -1 -1 -1 -1 -1 -1 -1
1 1 1 0 0 -1 -1 -1 -1 -1 -1 0 0 1 1 1
1 1 0 0 0 0 -1 -1 1 1 0 0 0 0 -1 -1
1 0 0 -1 -1 0 0 1 1 0 0 -1 -1 0 0 1
1 1 -1 -1 -1 -1 1 1 -1 -1 1 1 1 1 -1 -1
1 0 -1 -1 1 1 0 -1 -1 0 1 1 -1 -1 0 1
0 0 -1 1 1 -1 -1 1 -1 1 1 -1 -1 1 0 0
1 -1 -1 1 1 -1 -1 1 1 -1 -1 1 1 -1 -1 1
1 -1 -1 1 0 0 1 -1 1 -1 0 0 -1 1 1 -1
1 -1 0 1 -1 0 1 -1 -1 1 0 -1 1 0 -1 1
0 0 1 1 -1 -1 0 0 0 0 1 1 -1 -1 0 0
0 -1 1 0 0 1 -1 0 0 -1 1 0 0 1 -1 0
1 -1 1 -1 1 -1 0 0 0 0 1 -1 1 -1 1 -1
0 -1 1 -1 1 -1 1 0 0 1 -1 1 -1 1 -1 0
1 -1 0 0 -1 1 -1 1 -1 1 -1 1 0 0 1 -1
"""


def build_T() -> np.ndarray:
    """T of PAPER.md:270-287 as an int64 16x16 array (row-major as printed)."""
    rows = [[int(v) for v in line.split()] for line in _T_ROWS.strip().splitlines()]
    T = np.array(rows, dtype=np.int64)
    assert T.shape == (N, N)
    return T


def gram_diag(T: np.ndarray) -> np.ndarray:
    """diag(T·Tᵀ) — PAPER.md:296-304 states T·Tᵀ is diagonal; the diagonal
    is what S orthonormalises."""
    G = T @ T.T
    return np.diag(G).copy()


# S typed as printed: diag(1/4, 1/4, 1/√12, 1/√8, 1/√8, 1/4,
# 1/√12, 1/√12, 1/4, 1/√12, 1/√12, 1/√8, 1/√8, 1/√12, 1/√12, 1/√12).
_S_DENOMS_SQUARED = [16, 16, 12, 8, 8, 16, 12, 12, 16, 12, 12, 8, 8, 12, 12, 12]


def build_S_diag() -> np.ndarray:
    """Diagonal of S as printed at PAPER.md:315-329 (float64)."""
    return np.array([1.0 / math.sqrt(d) for d in _S_DENOMS_SQUARED], dtype=np.float64)


def build_C_hat() -> np.ndarray:
    """Ĉ = S·T, PAPER.md:305-313 (float64)."""
    return build_S_diag()[:, None] * build_T().astype(np.float64)


# --------------------------------------------------------------------------
# §2, Eq. (1), PAPER.md:347-469 — the sparse factorisation
# T = P2 · M4 · M3 · M2 · P1 · M1.
# --------------------------------------------------------------------------
def identity(n: int) -> np.ndarray:
    return np.eye(n, dtype=np.int64)


def counter_identity(n: int) -> np.ndarray:
    """Ī_n, the counter-identity of PAPER.md:467-469 (ones on the anti-diagonal)."""
    return np.fliplr(np.eye(n, dtype=np.int64))


def _butterfly(n: int) -> np.ndarray:
    """[[I_{n/2}, Ī_{n/2}], [Ī_{n/2}, -I_{n/2}]] as used by M1 and M2."""
    h = n // 2
    top = np.hstack([identity(h), counter_identity(h)])
    bot = np.hstack([counter_identity(h), -identity(h)])
    return np.vstack([top, bot])


def _block_diag(*blocks: np.ndarray) -> np.ndarray:
    n = sum(b.shape[0] for b in blocks)
    out = np.zeros((n, n), dtype=np.int64)
    o = 0
    for b in blocks:
        k = b.shape[0]
        out[o:o + k, o:o + k] = b
        o += k
    return out


def build_M1() -> np.ndarray:
    """M1 = [[I8, Ī8], [Ī8, -I8]]."""
    return _butterfly(16)


# P1 = diag(I9, 7x7 block), the block typed row by row.
_P1_BLOCK = """
0 0 1 0 0 0 0
0 0 0 1 0 0 0
0 0 0 0 0 0 1
0 0 0 0 0 1 0
0 0 0 0 1 0 0
0 1 0 0 0 0 0
1 0 0 0 0 0 0
"""


def build_P1() -> np.ndarray:
    """P1 = diag(I9, the printed 7x7 permutation)."""
    blk = np.array([[int(v) for v in l.split()] for l in _P1_BLOCK.strip().splitlines()],
                   dtype=np.int64)
    return _block_diag(identity(9), blk)


def build_M2() -> np.ndarray:
    """M2 = diag(B8, B8), B8 = [[I4, Ī4], [Ī4, -I4]]."""
    return _block_diag(_butterfly(8), _butterfly(8))


# the four 4x4 blocks of M3, typed as printed.
_M3_BLOCKS = [
    "1 0 0 1 / 0 1 1 0 / 0 -1 1 0 / 1 0 0 -1",
    "0 1 1 1 / -1 -1 0 1 / -1 1 -1 0 / 1 0 -1 1",
    "1 0 0 1 / 0 1 1 0 / 0 -1 1 0 / -1 0 0 1",
    "0 1 1 1 / 1 1 0 -1 / 1 -1 1 0 / 1 0 -1 1",
]


def build_M3() -> np.ndarray:
    """M3 = diag of the four printed 4x4 blocks."""
    blocks = []
    for s in _M3_BLOCKS:
        rows = [[int(v) for v in r.split()] for r in s.split("/")]
        blocks.append(np.array(rows, dtype=np.int64))
    return _block_diag(*blocks)


def build_M4() -> np.ndarray:
    """M4 = diag([[1,1],[1,-1]], I6, [[1,1],[1,-1]], I6)."""
    h = np.array([[1, 1], [1, -1]], dtype=np.int64)
    return _block_diag(h, identity(6), h, identity(6))


# "(0)(1 8)(2 4 3 11 10 7 12 2)(5 9 13 14 6 5)(15) in cyclic
# notation".  Reading A1: the repeated last element of a cycle
# marks its closure, so the cycles are (2 4 3 11 10 7 12) and (5 9 13 14 6).
P2_CYCLES_AS_PRINTED = "(0)(1 8)(2 4 3 11 10 7 12 2)(5 9 13 14 6 5)(15)"


def parse_cycles(text: str) -> list[int]:
    """Cycle notation -> sigma with sigma[i] = image of i (i -> next in cycle).

    Reading A1: a trailing repeat of the cycle's first element is the closure
    marker, not a new element.
    """
    sigma = list(range(N))
    for grp in text.replace(")", " ").split("("):
        elems = [int(v) for v in grp.split()]
        if not elems:
            continue
        if len(elems) > 1 and elems[-1] == elems[0]:
            elems = elems[:-1]
        for a, b in zip(elems, elems[1:] + elems[:1]):
            sigma[a] = b
    assert sorted(sigma) == list(range(N)), "not a permutation"
    return sigma


def build_P2(sigma: list[int] | None = None) -> np.ndarray:
    """P2 with (P2·e)_i = e_{sigma(i)}, sigma from PAPER.md:465 under reading A1."""
    if sigma is None:
        sigma = parse_cycles(P2_CYCLES_AS_PRINTED)
    P = np.zeros((N, N), dtype=np.int64)
    for i, s in enumerate(sigma):
        P[i, s] = 1
    return P


def factor_list() -> list[tuple[str, np.ndarray]]:
    """The stages in application order (right to left of Eq. (1))."""
    return [("M1", build_M1()), ("P1", build_P1()), ("M2", build_M2()),
            ("M3", build_M3()), ("M4", build_M4()), ("P2", build_P2())]


def factor_product() -> np.ndarray:
    """P2·M4·M3·M2·P1·M1 (exact int64)."""
    out = identity(N)
    for _, F in factor_list():
        out = F @ out
    return out


# --------------------------------------------------------------------------
# Staged (fast) evaluation with instrumented operation counting, Table 1
# (PAPER.md:526-548): "Proposed: 0 multiplications, 60 additions, 0 shifts".
# --------------------------------------------------------------------------
class OpCounter:
    def __init__(self) -> None:
        self.adds = 0
        self.mults = 0
        self.shifts = 0


class Counted:
    """An integer that counts every addition / subtraction it takes part in."""

    __slots__ = ("v", "c")

    def __init__(self, v: int, c: OpCounter) -> None:
        self.v = v
        self.c = c

    def __add__(self, o: "Counted") -> "Counted":
        self.c.adds += 1
        return Counted(self.v + o.v, self.c)

    def __sub__(self, o: "Counted") -> "Counted":
        self.c.adds += 1
        return Counted(self.v - o.v, self.c)

    def __neg__(self) -> "Counted":
        # A sign change of a lone term is absorbed by the following subtraction;
        # stage rows that are a single negated term do not occur in Eq. (1).
        return Counted(-self.v, self.c)


def apply_stage_counted(F: np.ndarray, x: list[Counted]) -> list[Counted]:
    """y = F·x evaluated row by row as a signed sum of the row's nonzero terms.

    A row with a single +1 is wiring (0 ops); a row with m nonzero ±1 terms costs
    m-1 additions/subtractions (started from a positive term when one exists).
    """
    y = []
    for row in F:
        terms = [(int(row[j]), x[j]) for j in range(len(row)) if row[j] != 0]
        assert all(abs(s) == 1 for s, _ in terms), "stage entries must be 0/±1"
        terms.sort(key=lambda t: -t[0])  # positive terms first
        s0, acc = terms[0]
        if s0 < 0:
            acc = -acc
        for s, v in terms[1:]:
            acc = acc + v if s > 0 else acc - v
        y.append(acc)
    return y


def fast_forward_1d(x, count: OpCounter | None = None, per_stage: dict | None = None):
    """y = T·x through the staged factorisation M1, P1, M2, M3, M4, P2.

    Returns a list of Python ints.  ``count`` accumulates the additions;
    ``per_stage`` (if given) receives the additions of each named stage.
    """
    c = count if count is not None else OpCounter()
    v = [Counted(int(a), c) for a in x]
    for name, F in factor_list():
        before = c.adds
        v = apply_stage_counted(F, v)
        if per_stage is not None:
            per_stage[name] = per_stage.get(name, 0) + (c.adds - before)
    return [a.v for a in v]


def fast_inverse_1d(y, count: OpCounter | None = None):
    """x = Tᵀ·y through the transposed stages M1ᵀ P1ᵀ M2ᵀ M3ᵀ M4ᵀ P2ᵀ applied
    in reverse order (the transposed signal-flow graph of Eq. (1))."""
    c = count if count is not None else OpCounter()
    v = [Counted(int(a), c) for a in y]
    for _, F in reversed(factor_list()):
        v = apply_stage_counted(F.T.copy(), v)
    return [a.v for a in v]


# --------------------------------------------------------------------------
# Reference transforms used by §3 and the config-5 sweep.
# --------------------------------------------------------------------------
def build_dct(n: int = N) -> np.ndarray:
    """Exact orthonormal DCT-II by brute-force cosines (reading A19):
    C[0][j] = sqrt(1/n), C[i][j] = sqrt(2/n)·cos(pi·i·(2j+1)/(2n))."""
    C = np.empty((n, n), dtype=np.float64)
    for i in range(n):
        a = math.sqrt(1.0 / n) if i == 0 else math.sqrt(2.0 / n)
        for j in range(n):
            C[i, j] = a * math.cos(math.pi * i * (2 * j + 1) / (2 * n))
    return C


def build_wht_natural(n: int = N) -> np.ndarray:
    """Sylvester (natural-order) Hadamard / sqrt(n).  Reading A15: natural order
    reproduces Table 2's WHT row."""
    H = np.array([[1]], dtype=np.float64)
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    return H / math.sqrt(n)


def markov_R(rho: float = 0.95, n: int = N) -> np.ndarray:
    """R[i,j] = rho^|i-j|, PAPER.md:684-694 (rho = 0.95)."""
    idx = np.arange(n)
    return rho ** np.abs(idx[:, None] - idx[None, :]).astype(np.float64)


def klt(rho: float = 0.95, n: int = N) -> np.ndarray:
    """KLT of R: eigenvectors as rows, descending eigenvalue."""
    w, V = np.linalg.eigh(markov_R(rho, n))
    order = np.argsort(w)[::-1]
    return V[:, order].T.copy()


def dct_distortion(Ct: np.ndarray, C: np.ndarray | None = None) -> float:
    """d2 = 1 - (1/N)·||diag(C·C̃ᵀ)||²."""
    C = build_dct() if C is None else C
    d = np.diag(C @ Ct.T)
    return 1.0 - float(np.sum(d * d)) / Ct.shape[0]


def total_error_energy(Ct: np.ndarray, C: np.ndarray | None = None) -> float:
    """epsilon = pi·||C - C̃||_F²."""
    C = build_dct() if C is None else C
    return math.pi * float(np.sum((C - Ct) ** 2))


def mse(Ct: np.ndarray, rho: float = 0.95, C: np.ndarray | None = None) -> float:
    """MSE = (1/N)·tr((C - C̃)·R·(C - C̃)ᵀ)."""
    C = build_dct() if C is None else C
    D = C - Ct
    return float(np.trace(D @ markov_R(rho, Ct.shape[0]) @ D.T)) / Ct.shape[0]


def coding_gain(Ct: np.ndarray, rho: float = 0.95) -> float:
    """C_g of PAPER.md:716-744 with s = C̃·R·C̃ᵀ."""
    n = Ct.shape[0]
    s = Ct @ markov_R(rho, n) @ Ct.T
    num = np.sum(np.diag(s)) / n
    prod_terms = np.diag(s) * np.sqrt(np.sum(Ct * Ct, axis=1))
    den = float(np.prod(prod_terms)) ** (1.0 / n)
    return 10.0 * math.log10(num / den)


def transform_efficiency(Ct: np.ndarray, rho: float = 0.95) -> float:
    """eta = sum|s_ii| / sum|s_ij| x 100."""
    s = Ct @ markov_R(rho, Ct.shape[0]) @ Ct.T
    return float(np.sum(np.abs(np.diag(s))) / np.sum(np.abs(s)) * 100.0)


def table2_row(Ct: np.ndarray) -> dict:
    """The five Table 2 measures for one transform."""
    return {"d2": dct_distortion(Ct), "eps": total_error_energy(Ct), "mse": mse(Ct),
            "cg": coding_gain(Ct), "eta": transform_efficiency(Ct)}


# --------------------------------------------------------------------------
# §4 zig-zag.  Reading A4: JPEG boustrophedon over the
# anti-diagonals d = 0..30 of the (row k, column l) grid, starting (0,0),(0,1),(1,0).
# --------------------------------------------------------------------------
def zigzag(n: int = N) -> list[tuple[int, int]]:
    order = []
    for d in range(2 * n - 1):
        cells = [(k, d - k) for k in range(n) if 0 <= d - k < n]  # k increasing
        if d % 2 == 0:
            cells = cells[::-1]  # even d: row decreasing (moving up-right)
        order.extend(cells)
    return order


def zonal_mask(r: int, n: int = N) -> np.ndarray:
    """M_r: 1 on the first r zig-zag positions, 0 elsewhere.
    Reading A18: r outside [1, 256] is a domain error."""
    if not (1 <= r <= n * n):
        raise ValueError(f"r={r} outside [1, {n * n}]")
    M = np.zeros((n, n), dtype=np.int64)
    for (k, l) in zigzag(n)[:r]:
        M[k, l] = 1
    return M
