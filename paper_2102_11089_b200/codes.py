"""Code graphs for the decode path: parity-check matrices, QC lifting,
puncturing and the edge-indexed Tanner layout the CUDA decoder consumes.

Mirrors the names and contracts of the reference's
``ldpc_ids.codes`` (/root/reference/pkg/src/ldpc_ids/codes.py) for the pieces
the decode path needs:

* ``ParityCheckMatrix`` / ``BaseGraph`` / ``CodeSpec`` validation  (codes.py:15-87)
* ``build_tanner`` edge numbering -- the tie-break contract      (codes.py:251-275)
* ``lift_base_graph`` / ``apply_puncture``                        (codes.py:225-248)
* ``make_random_regular_code`` (socket model, same RNG call order) (codes.py:337-372)
* ``syndrome_ok`` / ``graph_stats``                               (codes.py:278-301)

alist I/O and manifests are plumbing outside the decode path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class CodeError(ValueError):
    """Malformed code description (same role as reference codes.py:11)."""


@dataclass(frozen=True)
class ParityCheckMatrix:
    """Sparse binary H given by its one-entries (codes.py:15-37)."""

    m_rows: int
    n_cols: int
    entries: frozenset  # of (row, col)

    def __post_init__(self):
        if self.m_rows <= 0 or self.n_cols <= 0:
            raise CodeError("matrix dimensions must be positive")
        if not self.entries:
            raise CodeError("matrix has an empty row")
        arr = np.array(sorted(self.entries), dtype=np.int64).reshape(-1, 2)
        r, c = arr[:, 0], arr[:, 1]
        bad = (r < 0) | (r >= self.m_rows) | (c < 0) | (c >= self.n_cols)
        if bad.any():
            k = int(np.flatnonzero(bad)[0])
            raise CodeError(f"entry ({r[k]},{c[k]}) out of bounds "
                            f"{self.m_rows}x{self.n_cols}")
        if len(np.unique(r)) != self.m_rows:
            raise CodeError("matrix has an empty row")
        if len(np.unique(c)) != self.n_cols:
            raise CodeError("matrix has an empty column")

    @classmethod
    def from_arrays(cls, m_rows, n_cols, rows, cols):
        return cls(m_rows=int(m_rows), n_cols=int(n_cols),
                   entries=frozenset(zip(np.asarray(rows).tolist(),
                                         np.asarray(cols).tolist())))


@dataclass(frozen=True)
class BaseGraph:
    """Protograph with circulant shifts, -1 = zero block (codes.py:40-57)."""

    rows: int
    cols: int
    shifts: tuple
    lifting_size: int

    def __post_init__(self):
        if self.lifting_size <= 0:
            raise CodeError("lifting size must be positive")
        for r in range(self.rows):
            for c in range(self.cols):
                s = self.shifts[r][c]
                if s != -1 and not (0 <= s < self.lifting_size):
                    raise CodeError(
                        f"shift {s} at block ({r},{c}) outside [0,{self.lifting_size})")

    def to_text(self):
        """Reference base-graph text: 'rows cols Z' then the shift grid (codes.py:204-222)."""
        lines = [f"{self.rows} {self.cols} {self.lifting_size}"]
        lines += [" ".join(str(v) for v in row) for row in self.shifts]
        return "\n".join(lines) + "\n"


@dataclass(frozen=True)
class CodeSpec:
    """Matrix + puncture set + payload size (codes.py:60-87)."""

    h: ParityCheckMatrix
    punctured: tuple
    k_info: int
    label: str = ""

    def __post_init__(self):
        n = self.h.n_cols
        for p in self.punctured:
            if not 0 <= p < n:
                raise CodeError(f"punctured index {p} out of range")
        if len(set(self.punctured)) != len(self.punctured):
            raise CodeError("duplicate punctured indices")
        if self.k_info != n - self.h.m_rows:
            raise CodeError(
                f"k_info={self.k_info} inconsistent with N-M={n - self.h.m_rows}")

    @property
    def n_transmitted(self):
        return self.h.n_cols - len(self.punctured)

    @property
    def rate_tx(self):
        """K / (N - |punctured|) (codes.py:84-87)."""
        return self.k_info / self.n_transmitted


@dataclass
class TannerGraph:
    """Edge-indexed bipartite graph, edges in (check-major, vn-minor) order."""

    n_vars: int
    n_checks: int
    edge_cn: np.ndarray   # (E,) int64
    edge_vn: np.ndarray   # (E,) int64
    cn_ptr: np.ndarray    # (M+1,)
    vn_ptr: np.ndarray    # (N+1,)
    vn_edges: np.ndarray  # (E,) per-VN edge ids, ascending by check (= by edge id)
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def n_edges(self):
        return len(self.edge_cn)

    def vn_degree(self, n):
        return int(self.vn_ptr[n + 1] - self.vn_ptr[n])

    def cn_degree(self, m):
        return int(self.cn_ptr[m + 1] - self.cn_ptr[m])

    def vn_neighbors(self, n):
        es = self.vn_edges[self.vn_ptr[n]:self.vn_ptr[n + 1]]
        return [(int(self.edge_cn[e]), int(e)) for e in es]

    def cn_neighbors(self, m):
        return [(int(self.edge_vn[e]), int(e))
                for e in range(int(self.cn_ptr[m]), int(self.cn_ptr[m + 1]))]

    def edge_index(self, m, n):
        lo, hi = int(self.cn_ptr[m]), int(self.cn_ptr[m + 1])
        k = int(np.searchsorted(self.edge_vn[lo:hi], n))
        if k >= hi - lo or self.edge_vn[lo + k] != n:
            raise KeyError((m, n))
        return lo + k


def build_tanner(h):
    """Tanner graph of ``h`` with the reference's edge numbering.

    Edge ids follow sorted (check, vn) order (codes.py:257); ``vn_edges`` is a
    stable sort by VN so each VN's list ascends by check and by edge id
    (codes.py:269-270).  Every argmax tie-break in the decoder keys on these ids.
    """
    ent = np.array(sorted(h.entries), dtype=np.int64).reshape(-1, 2)
    edge_cn = np.ascontiguousarray(ent[:, 0])
    edge_vn = np.ascontiguousarray(ent[:, 1])
    cn_ptr = np.zeros(h.m_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(edge_cn, minlength=h.m_rows), out=cn_ptr[1:])
    vn_ptr = np.zeros(h.n_cols + 1, dtype=np.int64)
    np.cumsum(np.bincount(edge_vn, minlength=h.n_cols), out=vn_ptr[1:])
    vn_edges = np.argsort(edge_vn, kind="stable").astype(np.int64)
    return TannerGraph(n_vars=h.n_cols, n_checks=h.m_rows, edge_cn=edge_cn,
                       edge_vn=edge_vn, cn_ptr=cn_ptr, vn_ptr=vn_ptr,
                       vn_edges=vn_edges)


def lift_base_graph(bg):
    """Block (i,j) with shift s -> {(iZ+r, jZ+(r+s) mod Z)} (codes.py:225-240)."""
    z = bg.lifting_size
    rows, cols = [], []
    r = np.arange(z, dtype=np.int64)
    for i in range(bg.rows):
        for j in range(bg.cols):
            s = bg.shifts[i][j]
            if s == -1:
                continue
            rows.append(i * z + r)
            cols.append(j * z + (r + s) % z)
    return ParityCheckMatrix.from_arrays(bg.rows * z, bg.cols * z,
                                         np.concatenate(rows), np.concatenate(cols))


def parse_base_graph(text):
    """Parse 'rows cols Z' + shift grid (codes.py:204-222)."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise CodeError("base graph: empty input")
    head = lines[0].split()
    if len(head) != 3:
        raise CodeError("base graph line 1: expected 'rows cols Z'")
    rows, cols, z = (int(v) for v in head)
    if len(lines) != rows + 1:
        raise CodeError(f"base graph: expected {rows} shift rows, got {len(lines) - 1}")
    grid = []
    for i, ln in enumerate(lines[1:]):
        vals = [int(t) for t in ln.split()]
        if len(vals) != cols:
            raise CodeError(f"base graph line {i + 2}: expected {cols} values")
        grid.append(tuple(vals))
    return BaseGraph(rows=rows, cols=cols, shifts=tuple(grid), lifting_size=z)


def apply_puncture(h, prefix_len, k_info, label=""):
    """First ``prefix_len`` VNs never transmitted (codes.py:243-248)."""
    if prefix_len >= h.n_cols:
        raise CodeError(f"puncture prefix {prefix_len} >= N={h.n_cols}")
    return CodeSpec(h=h, punctured=tuple(range(prefix_len)), k_info=k_info, label=label)


def make_random_regular_code(n_vars, d_v, d_c, seed=0, label=None):
    """Seeded (d_v, d_c)-regular code, socket model (codes.py:337-372).

    Same generator, same draw order as the reference: one shuffle of the check
    sockets, then repeated repair passes that swap the first repeated socket
    with a uniformly drawn one.  Pinned by tests/test_codes.py against the
    reference's own output (edge-list digest).
    """
    if (n_vars * d_v) % d_c != 0:
        raise CodeError("n_vars * d_v must be divisible by d_c")
    m_rows = n_vars * d_v // d_c
    rng = np.random.default_rng(seed)
    vn_side = np.repeat(np.arange(n_vars), d_v)
    cn_side = np.repeat(np.arange(m_rows), d_c)
    rng.shuffle(cn_side)
    n_sock = len(vn_side)
    for _ in range(100 * n_sock):
        keys = cn_side.astype(np.int64) * n_vars + vn_side
        if len(np.unique(keys)) == n_sock:
            break
        # first socket whose (check, vn) pair already occurred earlier
        _, first = np.unique(keys, return_index=True)
        dup_mask = np.ones(n_sock, dtype=bool)
        dup_mask[first] = False
        i = int(np.flatnonzero(dup_mask)[0])
        j = int(rng.integers(n_sock))
        cn_side[i], cn_side[j] = cn_side[j], cn_side[i]
    else:
        raise CodeError("could not remove parallel edges; try another seed")
    h = ParityCheckMatrix.from_arrays(m_rows, n_vars, cn_side, vn_side)
    if label is None:
        label = f"random-{n_vars}-{d_v}-{d_c}-s{seed}"
    return CodeSpec(h=h, punctured=(), k_info=n_vars - m_rows, label=label)


def graph_stats(g):
    """E, mean degrees, degree histograms, degree-1 VN count (codes.py:278-291)."""
    vn_deg = np.diff(g.vn_ptr)
    cn_deg = np.diff(g.cn_ptr)
    return {
        "E": g.n_edges,
        "mean_vn_degree": g.n_edges / g.n_vars,
        "mean_cn_degree": g.n_edges / g.n_checks,
        "vn_degree_hist": dict(zip(*(a.tolist() for a in np.unique(vn_deg, return_counts=True)))),
        "cn_degree_hist": dict(zip(*(a.tolist() for a in np.unique(cn_deg, return_counts=True)))),
        "degree_one_vns": int((vn_deg == 1).sum()),
    }


def syndrome_ok(g, u_hat):
    """Every check has even parity over its neighbourhood (codes.py:294-301)."""
    u_hat = np.asarray(u_hat)
    if len(u_hat) != g.n_vars:
        raise CodeError(f"decision vector length {len(u_hat)} != N={g.n_vars}")
    sums = np.bincount(g.edge_cn, weights=u_hat[g.edge_vn].astype(np.int64),
                       minlength=g.n_checks)
    return bool((sums.astype(np.int64) % 2 == 0).all())
