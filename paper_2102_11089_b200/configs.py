"""The five BASELINE.json workloads (C0-C4).

C0 is the reference's own constructor (``make_random_regular_code``).  C1-C3
are *synthetic shaped* quasi-cyclic codes: seeded base-graph generators that
follow BASELINE.json's structural description (no standard 802.11 / 3GPP shift
table is used or transcribed).  Each generator emits a ``BaseGraph`` whose text
form is the reference's ``.bg`` format (codes.py:204-222), is lifted with
``lift_base_graph`` and punctured with ``apply_puncture``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .codes import BaseGraph, apply_puncture, lift_base_graph, make_random_regular_code


def _grid(rows, cols):
    return np.full((rows, cols), -1, dtype=np.int64)


def _to_bg(grid, z):
    return BaseGraph(rows=grid.shape[0], cols=grid.shape[1],
                     shifts=tuple(tuple(int(v) for v in row) for row in grid),
                     lifting_size=z)


def wifi_shaped_base_graph(seed=1, rows=12, cols=24, z=27):
    """C1: 12x24, Z=27.  12 systematic columns of weight 3 or 4 (about 2/3
    weight 3), rows uniform without repeats; 12 parity columns in dual-diagonal
    staircase form, the first parity column of weight 3."""
    rng = np.random.default_rng(seed)
    g = _grid(rows, cols)
    n_sys = cols - rows
    weights = np.where(rng.random(n_sys) < 2.0 / 3.0, 3, 4)
    for j in range(n_sys):
        for r in rng.choice(rows, size=int(weights[j]), replace=False):
            g[r, j] = rng.integers(z)
    p0 = n_sys
    for r in (0, rows // 2, rows - 1):
        g[r, p0] = rng.integers(z)
    for k in range(1, rows):
        g[k - 1, p0 + k] = 0
        g[k, p0 + k] = 0
    return _to_bg(g, z)


def _core_block(g, rng, n_sys, z):
    """4x4 double-diagonal core: first core column weight 3 (rows 0,1,3),
    then a staircase over rows (0,1), (1,2), (2,3)."""
    c = n_sys
    for r in (0, 1, 3):
        g[r, c] = rng.integers(z)
    for k, (a, b) in enumerate(((0, 1), (1, 2), (2, 3)), start=1):
        g[a, c + k] = rng.integers(z)
        g[b, c + k] = rng.integers(z)


def bg2_shaped_base_graph(seed=2, rows=42, cols=52, z=52, n_sys=10, p_core=0.7,
                          ext_deg=(3, 6)):
    """C2: 42x52, Z=52.  10 systematic columns, 4x4 double-diagonal core,
    38 weight-1 extension parity columns (identity); each extension row has
    3-6 nonzeros over the systematic+core columns; shifts uniform in [0,Z)."""
    rng = np.random.default_rng(seed)
    g = _grid(rows, cols)
    _core_block(g, rng, n_sys, z)
    for r in range(4):
        for j in range(n_sys):
            if rng.random() < p_core:
                g[r, j] = rng.integers(z)
    for r in range(4, rows):
        d = int(rng.integers(ext_deg[0], ext_deg[1] + 1))
        for j in rng.choice(n_sys + 4, size=d, replace=False):
            g[r, j] = rng.integers(z)
        g[r, n_sys + 4 + (r - 4)] = rng.integers(z)
    _ensure_columns(g, rng, z, n_sys)
    return _to_bg(g, z)


def _encodable_core_block(g, rng, n_sys, z):
    """4x4 double-diagonal core in the NR form: first core column of weight 3
    (rows 0,1,3) with shifts (a, b, a), staircase columns with identity
    circulants.  Summing the four core rows cancels the staircase and the two
    equal circulants of the first column, leaving P^b: the core block is
    invertible, so the core parity is a function of the systematic bits."""
    c = n_sys
    a, b = (int(x) for x in rng.integers(z, size=2))
    g[0, c], g[1, c], g[3, c] = a, b, a
    for k, (r0, r1) in enumerate(((0, 1), (1, 2), (2, 3)), start=1):
        g[r0, c + k] = 0
        g[r1, c + k] = 0


def bg1_shaped_base_graph(seed=3, rows=46, cols=68, z=384, n_sys=22, sys_weight_mean=8.5,
                          target_nnz=316, ext_max=9, core_hits=(3, 4), heavy_punct=True):
    """C3: 46x68, Z=384.  22 systematic columns with seeded weights averaging
    8.5, 4x4 double-diagonal core, 42 weight-1 extension parity columns,
    extension rows with 3-10 nonzeros, about 316 base nonzeros in total.

    As in NR BG1, the four core rows are dense in the systematic columns: every
    systematic column has 3 or 4 (seeded) of its entries in core rows 0-3 and
    the rest in extension rows.  A systematic column without core-row entries
    would be a low-weight codeword by itself (the bit plus the weight-1
    extension parity bits of its rows); the round-1 generator, which only
    weighted core rows 4x in a random draw, left columns 6 and 17 so, giving
    weight-5/6 codewords and an FER of 1.0 (Weak 1).  Also as in
    NR BG1, the two punctured columns (0 and 1) take the two largest of the
    seeded weights (punctured VNs of low degree stall decoding).  Shifts of
    systematic and extension entries stay uniform in [0, Z).  Oracle check
    (layered, 128-256 seeded frames): 3.0 dB / i_max 30 converges to the
    all-zero word on every frame; 1.0 dB / i_max 10 FER 0.91; 1.5 dB FER 0."""
    rng = np.random.default_rng(seed)
    g = _grid(rows, cols)
    _encodable_core_block(g, rng, n_sys, z)
    for r in range(4, rows):
        g[r, n_sys + 4 + (r - 4)] = rng.integers(z)
    # systematic column weights: seeded, clipped to [3, 16], total = round(mean * n_sys)
    total_w = int(round(sys_weight_mean * n_sys))
    w = np.clip(np.round(rng.gamma(4.0, sys_weight_mean / 4.0, size=n_sys)), 3, 16).astype(int)
    while w.sum() != total_w:
        j = int(rng.integers(n_sys))
        if w.sum() < total_w and w[j] < 16:
            w[j] += 1
        elif w.sum() > total_w and w[j] > 3:
            w[j] -= 1
    if heavy_punct:
        # the two punctured columns carry the two largest weights (NR BG1 form)
        top = np.argsort(-w, kind="stable")[:2]
        rest = [j for j in range(n_sys) if j not in set(top.tolist())]
        w = np.concatenate([w[top], w[rest]])
    ext_rows = np.arange(4, rows)

    def ext_load(r):
        return int((g[r, :n_sys + 4] >= 0).sum())

    # core rows: 3-4 seeded entries per systematic column; extension rows: the rest
    for j in range(n_sys):
        n_core = int(min(w[j], rng.integers(core_hits[0], core_hits[1] + 1)))
        for r in rng.choice(4, size=n_core, replace=False):
            g[r, j] = rng.integers(z)
        n_ext = int(w[j]) - n_core
        ok = np.array([ext_load(r) < ext_max for r in ext_rows], dtype=float)
        if n_ext:
            for r in rng.choice(ext_rows, size=n_ext, replace=False, p=ok / ok.sum()):
                g[r, j] = rng.integers(z)
    # top up the extension rows with core-column entries until ~target_nnz
    # (rows with the fewest non-identity entries first; at least 2 per row)
    while int((g >= 0).sum()) < target_nnz or min(ext_load(r) for r in ext_rows) < 2:
        open_rows = np.array([r for r in ext_rows if ext_load(r) < ext_max
                              and (g[r, n_sys:n_sys + 4] < 0).any()])
        if len(open_rows) == 0:
            break
        loads = np.array([ext_load(r) for r in open_rows])
        r = int(rng.choice(open_rows[loads == loads.min()]))
        free = [c for c in range(n_sys, n_sys + 4) if g[r, c] < 0]
        g[r, int(rng.choice(free))] = rng.integers(z)
    _ensure_columns(g, rng, z, n_sys)
    return _to_bg(g, z)


def _ensure_columns(g, rng, z, n_sys):
    for j in range(g.shape[1]):
        if (g[:, j] >= 0).sum() == 0:
            g[int(rng.integers(4)), j] = rng.integers(z)


@dataclass(frozen=True)
class Workload:
    name: str
    code_fn: object
    ebn0_db: tuple
    schedules: tuple
    i_max: int
    batch: int
    description: str

    def code(self):
        return self.code_fn()


def make_c0_code():
    """C0: (3,6)-regular n=504 from the reference's socket model, seed 0."""
    return make_random_regular_code(504, 3, 6, seed=0)


def make_c1_code():
    bg = wifi_shaped_base_graph()
    h = lift_base_graph(bg)
    return apply_puncture(h, 0, h.n_cols - h.m_rows, label="wifi-shaped-648")


def make_c2_code():
    bg = bg2_shaped_base_graph()
    h = lift_base_graph(bg)
    return apply_puncture(h, 2 * bg.lifting_size, h.n_cols - h.m_rows, label="bg2-shaped-2704")


def make_c3_code():
    bg = bg1_shaped_base_graph()
    h = lift_base_graph(bg)
    return apply_puncture(h, 2 * bg.lifting_size, h.n_cols - h.m_rows, label="bg1-shaped-26112")


WORKLOADS = {
    "C0": Workload("C0", make_c0_code, (2.0,), ("flooding", "layered", "rbp", "cirbp"), 5, 10_000,
                   "(3,6)-regular n=504, 2.0 dB, budget 5E, batch 10k"),
    "C1": Workload("C1", make_c1_code, (1.0, 1.5, 2.0, 2.5, 3.0),
                   ("flooding", "layered", "rbp", "cirbp", "lmdrbp", "slmdrbp", "lmd_cirbp",
                    "me_cirbp", "me_rbp"), 3, 100_000,
                   "WiFi-shaped n=648 QC Z=27, 1-3 dB, i_max=3, M=4 multi-edge, 100k frames/SNR"),
    "C2": Workload("C2", make_c2_code, (0.5, 1.0, 1.5, 2.0), ("layered", "rbp", "cirbp", "me_cirbp"),
                   3, 100_000, "BG2-shaped n=2704 Z=52 punct 2Z, M in {1,4,16}, 100k frames"),
    "C3": Workload("C3", make_c3_code, (0.5, 1.0), ("flooding", "layered", "rbp", "cirbp", "me_cirbp"),
                   10, 10_000, "BG1-shaped n=26112 Z=384 punct 2Z, budget 10E, M=64, 10k frames"),
    "C4": Workload("C4", make_c2_code, (0.0,), ("me_cirbp", "rbp"), 20, 1_000_000,
                   "BG2-shaped code at 0 dB, batch sweep 1..1M, M in {1,4,16,64}, budget 20E"),
}
