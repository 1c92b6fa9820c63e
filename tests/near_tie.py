"""Near-tie tracing of GPU-vs-oracle mismatches (north-star parity rule).

A frame whose GPU result differs from the CPU oracle is acceptable only if the
two update sequences first diverge at a selection the oracle logs as a
near-tie: relative top-2 gap (best - second) / max(best, 1e-8) < 1e-5 (the
floor is the float64 noise level of the +-30 messages; argmax ties; Alg.-4
group boundaries and
the n_p-th/(n_p+1)-th boundary for the multi-edge schedules, whose whole round
is chosen before its first update).  The GPU side comes from decode_batch_logged
(per-update propagated edge + committed C2V value), the oracle side from its
step log (oracle/ldpc_oracle.c, log_step / gap_note).
"""

import numpy as np
import torch

from oracle import pyoracle
from paper_2102_11089_b200.schedules import decode_batch_logged

NEAR_TIE = 1e-5


def trace(spec, g, llrs, cfg, frames, placement="auto", tol=NEAR_TIE):
    """Returns [(frame, divergence_step | None, oracle_gap | None, traced_bool)]."""
    frames = list(frames)
    if not frames:
        return []
    cap = int(min(cfg.i_max * g.n_edges + max(cfg.n_p, 1), 2_000_000))
    sub = np.ascontiguousarray(llrs[frames])
    out = decode_batch_logged(spec, torch.from_numpy(sub).cuda(), cfg, log_cap=cap, placement=placement)
    torch.cuda.synchronize()
    glog = out["step_log"].cpu().numpy()
    res = []
    for i, f in enumerate(frames):
        r = pyoracle.decode(g, sub[i].astype(np.float64), cfg.kind, cfg.kernel, cfg.i_max, spec.k_info,
                            cfg.gamma, cfg.n_p, cfg.n_g, cfg.selection_seed, log_cap=cap)
        ol, og = r["log_edge"], r["log_gap"]
        n = min(len(ol), cap)
        gl = glog[i][:n]
        bad = np.flatnonzero(gl != ol[:n])
        if len(bad) == 0:
            res.append((f, None, None, False))
            continue
        k = int(bad[0])
        # multi-edge rounds choose their whole set before the round's first
        # update, where the oracle logs that choice's gaps: look back one round
        w = cfg.n_p if cfg.kind.startswith("me_") else 1
        gap = float(og[max(0, k - w + 1):k + 1].min())
        res.append((f, k, gap, gap < tol))
    return res
