"""Generate golden vectors by running the REFERENCE decoder (this container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Imports ``ldpc_ids`` from /root/reference/pkg/src (read-only; never copied),
decodes seeded fp32-rounded BPSK-AWGN frames of the C0-C3 codes built by
paper_2102_11089_b200.configs with ``ldpc_ids.schedules.decode``
(schedules.py:111-158) and stores per-frame outputs in tests/golden/*.npz.
The CPU oracle (oracle/ldpc_oracle.c) must reproduce them bit-for-bit
(tests/test_oracle.py); the CUDA decoder is then checked against the oracle.
"""

from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))
REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent

from paper_2102_11089_b200 import configs, codes as mycodes  # noqa: E402
from paper_2102_11089_b200.channel import llr_batch  # noqa: E402


def _ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import ldpc_ids  # noqa: F401
    from ldpc_ids import codes, schedules
    return codes, schedules


def edge_digest(spec):
    g = mycodes.build_tanner(spec.h)
    return np.array([g.n_vars, g.n_checks, g.n_edges,
                     int(np.sum(g.edge_cn * 1_000_003 + g.edge_vn * 7) % (1 << 61))], np.int64)


def _ref_spec(spec):
    rc, _ = _ref()
    h = rc.ParityCheckMatrix(m_rows=spec.h.m_rows, n_cols=spec.h.n_cols, entries=spec.h.entries)
    return rc.CodeSpec(h=h, punctured=spec.punctured, k_info=spec.k_info, label=spec.label)


_SPEC_CACHE = {}


def _work(task):
    code_key, llrs, sched = task
    rc, rs = _ref()
    if code_key not in _SPEC_CACHE:
        spec = {"C0": configs.make_c0_code, "C1": configs.make_c1_code,
                "C2": configs.make_c2_code, "C3": configs.make_c3_code}[code_key]()
        rspec = _ref_spec(spec)
        _SPEC_CACHE[code_key] = (rspec, rc.build_tanner(rspec.h))
    rspec, graph = _SPEC_CACHE[code_key]
    cfg = rs.ScheduleConfig(**sched)
    res = []
    for row in llrs:
        r = rs.decode(rspec, row.astype(np.float64), cfg, graph=graph)
        c = r.counters
        res.append(dict(
            u_hat=np.packbits(r.u_hat), prop=int(r.iterations_used * graph.n_edges),
            converged=r.converged,
            counters=np.array([c.c2v_propagations, c.v2c_updates, c.c2v_pre_updates, c.ci_updates,
                               c.residual_ci_comparisons, c.multi_select_comparisons,
                               c.kappa_hits, c.kappa_trials], np.int64),
            biterr=np.asarray(r.bit_errors_at, np.int64),
            biterr_info=np.asarray(r.info_bit_errors_at, np.int64),
            kh=np.asarray(r.kappa_hits_iter, np.int64), kt=np.asarray(r.kappa_trials_iter, np.int64)))
    return res


def _stack(results):
    out = {}
    for k in results[0]:
        out[k] = np.stack([np.asarray(r[k]) for r in results])
    return out


def _tie_frames(n, rng):
    """Inputs engineered for exact ties: all-zero, quantised, saturated."""
    rows = [np.zeros(n), np.full(n, 30.0), np.full(n, 2.0)]
    q = rng.choice([-2.0, -1.0, 1.0, 2.0, 4.0], size=n, p=[0.1, 0.1, 0.3, 0.3, 0.2])
    rows.append(q)
    q2 = rng.choice([-1.0, 1.0, 3.0], size=n, p=[0.2, 0.5, 0.3])
    rows.append(q2)
    return np.array(rows, np.float32)


def plan():
    """(file, code, ebn0, n_frames, extra_rows, [schedule configs])"""
    ref8 = ["flooding", "rbp", "cirbp", "lmdrbp", "slmdrbp", "lmd_cirbp", "me_cirbp", "me_lmd_cirbp"]
    cases = []
    c0 = [dict(kind=k, i_max=5, n_p=4) for k in ref8]
    c0 += [dict(kind=k, i_max=5, kernel="minsum", n_p=4) for k in ref8]
    c0 += [dict(kind="me_cirbp", i_max=5, n_p=16), dict(kind="me_cirbp", i_max=5, n_p=1),
           dict(kind="me_lmd_cirbp", i_max=5, n_p=16, n_g=8, selection_seed=12345),
           dict(kind="cirbp", i_max=5, gamma=0.0), dict(kind="cirbp", i_max=5, gamma=0.5)]
    c0 += [dict(kind=k, i_max=0, n_p=4) for k in ref8] + [dict(kind=k, i_max=1, n_p=4) for k in ref8]
    cases.append(("c0", "C0", 2.0, 40, True, c0))
    cases.append(("c1", "C1", 2.0, 24, True, [dict(kind=k, i_max=3, n_p=4) for k in ref8]))
    c2 = [dict(kind=k, i_max=3, n_p=4) for k in ref8] + [dict(kind="me_cirbp", i_max=3, n_p=16)]
    cases.append(("c2", "C2", 1.0, 6, True, c2))
    # C3 at BASELINE configs[3]'s own budget (i_max 10) and both of its SNRs
    c3 = [dict(kind=k, i_max=10, n_p=64) for k in ("flooding", "rbp", "cirbp", "me_cirbp")]
    c3 += [dict(kind="lmd_cirbp", i_max=2), dict(kind="rbp", i_max=2, kernel="minsum")]
    cases.append(("c3", "C3", 1.0, 16, False, c3))
    cases.append(("c3b", "C3", 0.5, 16, False, c3[:4]))
    return cases


def _trace_work(task):
    code_key, llrs, sched = task
    rc, rs = _ref()
    spec = {"C0": configs.make_c0_code}[code_key]()
    rspec = _ref_spec(spec)
    graph = rc.build_tanner(rspec.h)
    cfg = rs.ScheduleConfig(**sched)
    return [np.asarray(rs.decode(rspec, row.astype(np.float64), cfg, graph=graph,
                                 want_trace=True).trace_llrs, np.float64) for row in llrs]


def make_trace_golden():
    """trace.npz: want_trace outputs (schedules.py:57, E:192-217, E:768-782) of
    the reference on C0 -- full arrays for frame 0, sha256 digests of every
    frame -- and J(gamma) counts of sim.mc_j_gamma (sim.py:339-353)."""
    import hashlib
    _ref()
    from ldpc_ids import sim as rsim, schedules as rs
    rc, _ = _ref()
    spec = configs.make_c0_code()
    rng = np.random.default_rng(11089)
    llrs = llr_batch(spec, 1.5, seed=0, start=0, count=5, dtype=np.float32)
    llrs = np.concatenate([llrs, _tie_frames(spec.h.n_cols, rng)[3:]])
    ref8 = ["flooding", "rbp", "cirbp", "lmdrbp", "slmdrbp", "lmd_cirbp", "me_cirbp", "me_lmd_cirbp"]
    scheds = [dict(kind=k, i_max=3, n_p=4) for k in ref8] + [dict(kind="rbp", i_max=3, kernel="minsum")]
    payload = {"llrs": llrs, "digest": edge_digest(spec), "schedules": np.array([repr(x) for x in scheds])}
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as pool:
        futs = [pool.submit(_trace_work, ("C0", llrs, sc)) for sc in scheds]
        for si, f in enumerate(futs):
            tr = f.result()
            payload[f"s{si}_trace0"] = tr[0]
            payload[f"s{si}_sha"] = np.array([hashlib.sha256(np.ascontiguousarray(t).tobytes()).hexdigest()
                                              for t in tr])
    rspec = _ref_spec(spec)
    gam = [0.0, 0.02, 0.1, 0.3, 0.6]
    jc = []
    jcases = [dict(kind="cirbp", i_max=3), dict(kind="rbp", i_max=3), dict(kind="flooding", i_max=3),
              dict(kind="me_cirbp", i_max=3, n_p=4)]
    for jc_cfg in jcases:
        r = rsim.mc_j_gamma(rspec, rs.ScheduleConfig(**jc_cfg), 1.0, gam, 96, master_seed=7)
        jc.append(np.asarray(r["counts"], np.int64))
    payload["j_gammas"] = np.array(gam)
    payload["j_cases"] = np.array([repr(x) for x in jcases])
    payload["j_counts"] = np.stack(jc)
    payload["j_ebn0"] = np.float64(1.0)
    payload["j_frames"] = np.int64(96)
    payload["j_seed"] = np.int64(7)
    np.savez_compressed(OUT / "trace.npz", **payload)


def make_sim_golden():
    """sim.npz: CSV records of the reference harness (sim.run_fer_sweep,
    sim.py:303-316) for a small C0 campaign -- block order, min_frame_errors
    stopping, per-iteration FER/BER, kappa per iteration."""
    _ref()
    from ldpc_ids import sim as rsim, schedules as rs
    spec = configs.make_c0_code()
    rspec = _ref_spec(spec)
    scheds = [dict(kind="cirbp", i_max=3), dict(kind="rbp", i_max=2), dict(kind="flooding", i_max=4),
              dict(kind="me_cirbp", i_max=3, n_p=4), dict(kind="lmdrbp", i_max=3, kernel="minsum")]
    camp = rsim.Campaign(code=rspec, schedules=[rs.ScheduleConfig(**x) for x in scheds],
                         snr_grid=[1.0, 2.0], min_frame_errors=12, max_frames=1500, master_seed=3)
    recs = rsim.run_fer_sweep(camp)
    csv_text = rsim.records_to_csv(recs)
    kp = [str(r.kappa_per_iteration) for r in recs]
    np.savez_compressed(OUT / "sim.npz", csv=np.array(csv_text), schedules=np.array([repr(x) for x in scheds]),
                        snr=np.array([1.0, 2.0]), min_frame_errors=np.int64(12), max_frames=np.int64(1500),
                        seed=np.int64(3), kappa_per_iteration=np.array(kp),
                        frame_errors_at=np.array([str(r.frame_errors_at) for r in recs]),
                        bit_errors_at=np.array([str(r.bit_errors_at) for r in recs]))


def _steps_work(task):
    """One frame through the reference's stepwise DecoderState (kernels.py:98-181):
    residual-argmax edge choice (lowest index among ties, like _decode_rbp),
    propagate(edge) for `steps` updates; returns the edge sequence, the committed
    C2V value of each update, the state after the last update and the
    recompute_all audit of that state."""
    code_key, llr, steps, kernel = task
    rc, rs = _ref()
    from ldpc_ids import kernels as rk
    spec = {"C0": configs.make_c0_code, "C1": configs.make_c1_code, "C2": configs.make_c2_code}[code_key]()
    rspec = _ref_spec(spec)
    graph = rc.build_tanner(rspec.h)
    st = rk.DecoderState(graph, np.asarray(llr, np.float64), kernel=kernel, maintain_ci=True)
    edges, vals = [], []
    for _ in range(steps):
        e = int(np.argmax(st.residual))  # first maximum = lowest edge id
        st.propagate(e)
        edges.append(e)
        vals.append(float(st.c2v[e]))
    res, total, pre_total, ci = st.recompute_all()
    c = st.counters
    return dict(edges=np.array(edges, np.int32), c2v=np.array(vals),
                s_c2v=st.c2v.copy(), s_pre=st.pre_c2v.copy(), s_total=st.total_llr.copy(),
                s_pretot=st.pre_total_llr.copy(), s_ci=st.ci.copy(),
                a_res=res, a_total=total, a_pretot=pre_total, a_ci=ci,
                counters=np.array([c.c2v_propagations, c.v2c_updates, c.c2v_pre_updates, c.ci_updates,
                                   c.residual_ci_comparisons, c.multi_select_comparisons, c.kappa_hits,
                                   c.kappa_trials], np.int64))


def make_steps_golden():
    """steps.npz: per-update traces of the reference's DecoderState.propagate
    (kernels.py:145-156) for the first 1000 updates of C0-C2 frames (exact and
    min-sum), with the final state and its recompute_all audit (kernels.py:161-181)."""
    _ref()
    cases = [("C0", 2.0, 4, "exact"), ("C1", 2.0, 3, "exact"), ("C2", 1.0, 2, "exact"), ("C0", 2.0, 2, "minsum"),
             ("C0", 6.0, 2, "exact"), ("C2", 5.0, 1, "exact")]
    payload = {}
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as pool:
        for ci_, (key, eb, nfr, kernel) in enumerate(cases):
            spec = {"C0": configs.make_c0_code, "C1": configs.make_c1_code, "C2": configs.make_c2_code}[key]()
            llrs = llr_batch(spec, eb, seed=0, start=500, count=nfr, dtype=np.float32)
            res = list(pool.map(_steps_work, [(key, l, 1000, kernel) for l in llrs]))
            payload[f"c{ci_}_case"] = np.array(repr(dict(code=key, ebn0=eb, kernel=kernel)))
            payload[f"c{ci_}_llrs"] = llrs
            for k in res[0]:
                payload[f"c{ci_}_{k}"] = np.stack([r[k] for r in res])
    payload["n_cases"] = np.int64(len(cases))
    np.savez_compressed(OUT / "steps.npz", **payload)


def main():
    if "--only-steps" in sys.argv:
        make_steps_golden()
        return
    if "--only-trace" in sys.argv:
        make_trace_golden()
        return
    if "--only-sim" in sys.argv:
        make_sim_golden()
        return
    t0 = time.time()
    _ref()
    rc, _ = _ref()
    # pin our restated make_random_regular_code against the reference's
    ref_c0 = rc.make_random_regular_code(504, 3, 6, seed=0)
    mine = configs.make_c0_code()
    assert ref_c0.h.entries == mine.h.entries, "C0 constructor drifted from the reference"
    rng = np.random.default_rng(2102_11089)
    only = sys.argv[sys.argv.index("--only") + 1].split(",") if "--only" in sys.argv else None
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as pool:
        for fname, key, ebn0, nfr, ties, scheds in plan():
            if only and fname not in only:
                continue
            spec = {"C0": configs.make_c0_code, "C1": configs.make_c1_code,
                    "C2": configs.make_c2_code, "C3": configs.make_c3_code}[key]()
            llrs = llr_batch(spec, ebn0, seed=0, start=0, count=nfr, dtype=np.float32)
            if ties:
                llrs = np.concatenate([llrs, _tie_frames(spec.h.n_cols, rng)])
            payload = {"llrs": llrs, "digest": edge_digest(spec), "ebn0": np.float64(ebn0)}
            futs = []
            for si, s in enumerate(scheds):
                chunks = np.array_split(np.arange(len(llrs)), min(len(llrs), os.cpu_count()))
                futs.append([pool.submit(_work, (key, llrs[c], s)) for c in chunks if len(c)])
            names = []
            for si, (s, fl) in enumerate(zip(scheds, futs)):
                res = [r for f in fl for r in f.result()]
                st = _stack(res)
                tag = f"s{si}"
                names.append(repr(s))
                for k, v in st.items():
                    payload[f"{tag}_{k}"] = v
            payload["schedules"] = np.array(names)
            np.savez_compressed(OUT / f"{fname}.npz", **payload)
            print(f"{fname}: {len(scheds)} schedules x {len(llrs)} frames  ({time.time() - t0:.0f}s)",
                  flush=True)
    if only:
        return
    # KATs (SPEC.md examples, evaluated by the reference)
    from ldpc_ids import kernels as rk, schedules as rs, _engine as re_
    kat = {}
    kat["c2v_22"] = rk.c2v_message([2.0, 2.0])
    kat["c2v_minsum"] = rk.c2v_message([2.0, -3.0], "minsum")
    kat["c2v_zero"] = rk.c2v_message([0.0, 5.0])
    sel, cmp_ = rs.select_vns([0.9, 0.7, 0.3, 0.1], 4, 2, 0)
    kat["select_vns_spec"] = sel
    ci = np.random.default_rng(7).random(300)
    for n_g, n_p, seed in ((16, 4, 0), (16, 64, 3), (4, 100, 99), (1, 10, 5), (64, 7, 2**63 + 11)):
        kat[f"select_{n_g}_{n_p}_{seed}"] = rs.select_vns(ci, n_g, n_p, seed)[0]
    kat["select_ci"] = ci
    seq = []
    for seed in (0, 1, 12345, -1, 2**62):
        st = np.array([seed], np.int64)
        seq.append([re_._rand_next(st) for _ in range(8)])
    kat["rand_seq"] = np.array(seq, np.int64)
    kat["p0_ln3"] = rk.posterior_p0(np.log(3.0))
    np.savez_compressed(OUT / "kat.npz", **{k: np.asarray(v) for k, v in kat.items()})
    make_trace_golden()
    make_sim_golden()
    print(f"done in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
