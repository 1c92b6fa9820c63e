"""Decoder API -- the drop-in for ``ldpc_ids.schedules`` on B200.

Same names, arguments, validation messages and result type as the reference
(/root/reference/pkg/src/ldpc_ids/schedules.py:20-193):

* ``ScheduleConfig`` (schedules.py:24-44), extended with the two schedules
  the reference lacks (``layered``, ``me_rbp``) and a ``precision`` field;
* ``decode(code, channel_llrs, config, graph=None, want_trace=False)``
  returning ``DecodeResult`` (schedules.py:47-57, 111-158);
* ``decode_<kind>`` wrappers that assert the kind (schedules.py:161-193);
* ``select_vns(ci, n_g, n_p, seed, search_set)`` (schedules.py:60-79);

plus ``decode_batch`` -- the call the B200 build is designed around: B frames
of LLRs (torch tensor on the GPU, or host array) decoded by one launch of the
sm_100a kernels through the C ABI.  Every call runs on the GPU; there is no
CPU path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np
import torch

from . import _native
from .codes import CodeSpec, TannerGraph, build_tanner
from .kernels import KERNELS, Counters

SCHEDULE_KINDS = ("flooding", "rbp", "cirbp", "lmdrbp", "slmdrbp", "lmd_cirbp", "me_cirbp",
                  "me_lmd_cirbp", "layered", "me_rbp")
KIND_IDS = {k: i for i, k in enumerate(SCHEDULE_KINDS)}
PRECISIONS = {"f64": 0, "f32": 1}


@dataclass(frozen=True)
class ScheduleConfig:
    kind: str
    gamma: float = 0.1
    n_p: int = 1
    n_g: int = 16
    i_max: int = 3
    kernel: str = "exact"
    selection_seed: int = 0
    precision: str = "f64"

    def __post_init__(self):
        if self.kind not in SCHEDULE_KINDS:
            raise ValueError(f"unknown schedule kind {self.kind!r}")
        if not 0.0 <= self.gamma < 1.0:
            raise ValueError("gamma must lie in [0, 1)")
        if self.n_p < 1 or self.n_g < 1:
            raise ValueError("n_p and n_g must be >= 1")
        if self.i_max < 0:
            raise ValueError("i_max must be >= 0")
        if self.kernel not in KERNELS:
            raise ValueError(f"unknown kernel {self.kernel!r}")
        if self.precision not in PRECISIONS:
            raise ValueError(f"unknown precision {self.precision!r}")


@dataclass
class DecodeResult:
    u_hat: np.ndarray
    converged: bool
    iterations_used: Fraction
    counters: Counters
    bit_errors_at: np.ndarray
    info_bit_errors_at: np.ndarray
    kappa_hits_iter: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    kappa_trials_iter: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    trace_llrs: np.ndarray | None = None


# ----------------------------------------------------------------- graph


class DeviceGraph:
    """Device-resident Tanner graph handle (ldpc_graph_create) on one GPU."""

    def __init__(self, g: TannerGraph, device=None):
        L = _native.lib()
        arrs = [np.ascontiguousarray(a, dtype=np.int32)
                for a in (g.edge_cn, g.edge_vn, g.cn_ptr, g.vn_ptr, g.vn_edges)]
        self._keep = arrs
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        h = C.c_void_p()
        with torch.cuda.device(self.device):  # the handle's arrays live on this device
            _native.check(L.ldpc_graph_create(*[a.ctypes.data_as(C.c_void_p) for a in arrs],
                                              g.n_vars, g.n_checks, g.n_edges, C.byref(h)),
                          "ldpc_graph_create")
        self.handle = h
        info = np.zeros(7, np.int64)
        L.ldpc_graph_info(h, info.ctypes.data_as(C.c_void_p))
        self.N, self.M, self.E, self.max_dv, self.max_dc, self.max_two_hop, self.n_levels = \
            (int(v) for v in info)
        self._ws = {}

    def __del__(self):
        try:
            if self.handle:
                _native.lib().ldpc_graph_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def workspace(self, sched, B, stream):
        """Scratch for one decode, cached per stream: decodes on different
        streams never share state, and a buffer is allocated on the stream
        that uses it, so the caching allocator only recycles it after the
        work queued there (the C ABI's stream-ordered contract)."""
        L = _native.lib()
        sz = C.c_size_t()
        _native.check(L.ldpc_workspace_size(self.handle, C.byref(sched), int(B), C.byref(sz)),
                      "ldpc_workspace_size")
        key = stream.cuda_stream
        ws = self._ws.get(key)
        if ws is None or ws.numel() < sz.value:
            self._ws.pop(key, None)
            with torch.cuda.stream(stream):
                ws = torch.empty(max(sz.value, 256), dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws


def _tanner_of(code: CodeSpec) -> TannerGraph:
    """The TannerGraph of a CodeSpec, cached on the (frozen) object itself so
    it lives exactly as long as the code does."""
    g = code.__dict__.get("_b200_tanner")
    if g is None:
        g = build_tanner(code.h)
        object.__setattr__(code, "_b200_tanner", g)
    return g


def device_graph(code_or_graph, device=None):
    """Cached DeviceGraph of a CodeSpec / TannerGraph on `device` (default: current)."""
    g = code_or_graph
    if isinstance(g, CodeSpec):
        g = _tanner_of(g)
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    per_dev = g._cache.setdefault("device", {})
    dg = per_dev.get(device.index)
    if dg is None:
        dg = DeviceGraph(g, device)
        per_dev[device.index] = dg
    return dg


PLACEMENTS = {"auto": 0, "hbm": 1, "split": 2, "smem": 3, "trees": 4}


def _sched(config: ScheduleConfig, k_info: int, llr_f64: bool, max_resident=0, placement="auto",
           want_trace=False, variant=0):
    seed = int(config.selection_seed) & 0xFFFFFFFFFFFFFFFF
    if seed >= 1 << 63:
        seed -= 1 << 64
    return _native.LdpcSched(KIND_IDS[config.kind], KERNELS[config.kernel], config.i_max,
                             config.n_p, config.n_g, int(k_info), float(config.gamma), seed,
                             PRECISIONS[config.precision], 1 if llr_f64 else 0,
                             int(max_resident), PLACEMENTS[placement], 1 if want_trace else 0,
                             _native.variant_bits(variant) if not isinstance(variant, int) else variant)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def decode_batch(code, llrs, config: ScheduleConfig, graph=None, k_info=None, device=None,
                 stream=None, out=None, max_resident=0, placement="auto", force_global=False,
                 want_trace=False, gammas=None, j_counts=None, variant=0):
    """Decode a batch of frames on the GPU.

    code: CodeSpec (k_info taken from it) or TannerGraph (pass k_info).
    llrs: [B, N] float32/float64 torch tensor (device or host) or numpy array.
    Returns a dict of device tensors: u_hat [B,N] int8, prop [B] int64,
    converged [B] bool, counters [B,8] int64, bit_errors_at / info_bit_errors_at
    [B, i_max+1] int32, kappa_hits_iter / kappa_trials_iter [B, i_max] int32.
    Asynchronous on the current (or given) stream.  placement (dynamic
    schedules): "auto", "smem", "split" (per-edge state in HBM/L2, per-VN
    state in shared memory) or "hbm".  variant: engine pin for tests and
    measurement (names of _native.VARIANTS, comma-separated; default: tuned).
    """
    if isinstance(code, CodeSpec):
        spec = code
        k_info = code.k_info if k_info is None else k_info
    else:
        spec = None
        if k_info is None:
            raise ValueError("k_info is required when decoding from a TannerGraph")
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    dg = device_graph(graph if graph is not None else code, device)
    if not torch.is_tensor(llrs):
        llrs = torch.from_numpy(np.ascontiguousarray(llrs))
    if llrs.dtype not in (torch.float32, torch.float64):
        llrs = llrs.to(torch.float64)
    if llrs.dim() != 2 or llrs.shape[1] != dg.N:
        raise ValueError("channel LLR length mismatch")
    llrs = llrs.to(device, non_blocking=True).contiguous()
    if config.kind in ("me_cirbp", "me_lmd_cirbp") and config.n_p > dg.N:
        raise ValueError("n_p exceeds the number of variable nodes")
    B = llrs.shape[0]
    I = config.i_max
    if force_global:
        placement = "hbm"
    tracing = bool(want_trace) or gammas is not None
    sched = _sched(config, k_info, llrs.dtype == torch.float64, max_resident, placement, tracing, variant)
    st = stream if stream is not None else torch.cuda.current_stream(device)
    with torch.cuda.device(device), torch.cuda.stream(st):
        return _decode_on(dg, llrs, B, I, sched, config, device, st, out, tracing, want_trace, gammas,
                          j_counts)


def _decode_on(dg, llrs, B, I, sched, config, device, st, out, tracing, want_trace, gammas, j_counts):
    if out is None:
        out = {
            "u_hat": torch.empty((B, dg.N), dtype=torch.int8, device=device),
            "prop": torch.empty(B, dtype=torch.int64, device=device),
            "converged": torch.empty(B, dtype=torch.uint8, device=device),
            "counters": torch.empty((B, 8), dtype=torch.int64, device=device),
            "bit_errors_at": torch.empty((B, I + 1), dtype=torch.int32, device=device),
            "info_bit_errors_at": torch.empty((B, I + 1), dtype=torch.int32, device=device),
            "kappa_hits_iter": torch.zeros((B, max(I, 1)), dtype=torch.int32, device=device),
            "kappa_trials_iter": torch.zeros((B, max(I, 1)), dtype=torch.int32, device=device),
        }
    ws = dg.workspace(sched, B, st)
    L = _native.lib()
    if not tracing:
        rc = L.ldpc_decode(dg.handle, _ptr(llrs), B, C.byref(sched), _ptr(out["u_hat"]), _ptr(out["prop"]),
                           _ptr(out["converged"]), _ptr(out["counters"]), _ptr(out["bit_errors_at"]),
                           _ptr(out["info_bit_errors_at"]), _ptr(out["kappa_hits_iter"]),
                           _ptr(out["kappa_trials_iter"]), _ptr(ws), ws.numel(),
                           C.c_void_p(st.cuda_stream))
        _native.check(rc, "ldpc_decode")
    else:
        trace = None
        if want_trace and want_trace != "counts":
            trace = torch.empty((B, I + 1, 2 * dg.N), dtype=torch.float64, device=device)
            out["trace_llrs"] = trace
        gam = None
        if gammas is not None:
            gam = torch.as_tensor(np.asarray(list(gammas), np.float64), device=device)
            if gam.numel() < 1:
                raise ValueError("gammas must be non-empty")
            if j_counts is None:
                j_counts = torch.zeros((I + 1, gam.numel(), 2), dtype=torch.int64, device=device)
            out["j_counts"] = j_counts
        rc = L.ldpc_decode_traced(dg.handle, _ptr(llrs), B, C.byref(sched), _ptr(out["u_hat"]),
                                  _ptr(out["prop"]), _ptr(out["converged"]), _ptr(out["counters"]),
                                  _ptr(out["bit_errors_at"]), _ptr(out["info_bit_errors_at"]),
                                  _ptr(out["kappa_hits_iter"]), _ptr(out["kappa_trials_iter"]),
                                  _ptr(trace), _ptr(gam), 0 if gam is None else gam.numel(),
                                  _ptr(j_counts), _ptr(ws), ws.numel(), C.c_void_p(st.cuda_stream))
        _native.check(rc, "ldpc_decode_traced")
    out["_launches"] = L.ldpc_last_launch_count()
    return out


def results_to_numpy(out, kind, i_max):
    r = {k: v.cpu().numpy() for k, v in out.items() if torch.is_tensor(v)}
    r["converged"] = r["converged"].astype(bool)
    r["kappa_hits_iter"] = r["kappa_hits_iter"][:, :i_max]
    r["kappa_trials_iter"] = r["kappa_trials_iter"][:, :i_max]
    return r


def decode(code: CodeSpec, channel_llrs, config: ScheduleConfig, graph=None,
           want_trace=False) -> DecodeResult:
    """Run one frame through the configured schedule (schedules.py:111-158)."""
    if graph is None:
        graph = _tanner_of(code)
    chl = np.asarray(channel_llrs, dtype=np.float64)
    if chl.ndim != 1 or len(chl) != graph.n_vars:
        raise ValueError("channel LLR length mismatch")
    out = decode_batch(graph, chl[None, :], config, k_info=code.k_info, want_trace=bool(want_trace))
    r = results_to_numpy(out, config.kind, config.i_max)
    kh = kt = np.zeros(0, np.int64)
    if config.kind == "cirbp":
        kh = r["kappa_hits_iter"][0].astype(np.int64)
        kt = r["kappa_trials_iter"][0].astype(np.int64)
    return DecodeResult(
        u_hat=r["u_hat"][0].astype(np.int8),
        converged=bool(r["converged"][0]),
        iterations_used=Fraction(int(r["prop"][0]), graph.n_edges),
        counters=Counters.from_array(r["counters"][0]),
        bit_errors_at=r["bit_errors_at"][0].astype(np.int64),
        info_bit_errors_at=r["info_bit_errors_at"][0].astype(np.int64),
        kappa_hits_iter=kh, kappa_trials_iter=kt,
        trace_llrs=r["trace_llrs"][0] if want_trace else None)


def select_vns(ci_values, n_g, n_p, seed, search_set=None):
    """Algorithm-4 group selection on the GPU (schedules.py:60-79)."""
    ci = np.ascontiguousarray(ci_values, dtype=np.float64)
    mask = np.zeros(len(ci), dtype=np.uint8)
    if search_set is None:
        mask[:] = 1
    else:
        mask[np.asarray(list(search_set), dtype=np.int64)] = 1
    if mask.sum() < n_p:
        raise ValueError("search set smaller than n_p")
    dev = torch.device("cuda", torch.cuda.current_device())
    ci_d = torch.from_numpy(ci).to(dev)
    mask_d = torch.from_numpy(mask).to(dev)
    out = torch.zeros(n_p, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    s = int(seed) & 0xFFFFFFFFFFFFFFFF
    if s >= 1 << 63:
        s -= 1 << 64
    L = _native.lib()
    _native.check(L.ldpc_select_vns(_ptr(ci_d), _ptr(mask_d), len(ci), n_g, n_p, s, _ptr(out),
                                    _ptr(cnt), C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)),
                  "ldpc_select_vns")
    k = int(cnt.item())
    return out[:k].cpu().numpy().astype(np.int64), n_g


def _wrap(kinds):
    def fn(code, channel_llrs, config, **kw):
        assert config.kind in kinds
        return decode(code, channel_llrs, config, **kw)
    return fn


decode_flooding = _wrap(("flooding",))
decode_rbp = _wrap(("rbp",))
decode_cirbp = _wrap(("cirbp",))
decode_lmdrbp = _wrap(("lmdrbp", "slmdrbp"))
decode_lmd_cirbp = _wrap(("lmd_cirbp",))
decode_me_cirbp = _wrap(("me_cirbp",))
decode_me_lmd_cirbp = _wrap(("me_lmd_cirbp",))
decode_layered = _wrap(("layered",))
decode_me_rbp = _wrap(("me_rbp",))


def decode_replay(code, llrs, forced_edges, kernel="exact", precision="f64", k_info=None, stream=None):
    """The GPU side of the reference's stepwise DecoderState (kernels.py:98-181):
    each frame is initialised like every schedule (_init_state) and then
    propagates the GIVEN edges forced_edges[B, steps] (pre_total and CI
    maintained, like DecoderState(maintain_ci=True)) through ldpc_decode_replay.
    Returns device tensors: c2v_trace [B, steps] float64 (the value each update
    commits), c2v / pre_c2v [B, E], total / pre_total / ci [B, N] float64 (the
    state recompute_all audits) and counters [B, 8] int64."""
    if isinstance(code, CodeSpec):
        k_info = code.k_info if k_info is None else k_info
    dev = torch.device("cuda", torch.cuda.current_device())
    dg = device_graph(code, dev)
    if not torch.is_tensor(llrs):
        llrs = torch.from_numpy(np.ascontiguousarray(llrs))
    llrs = llrs.to(dev).contiguous()
    if llrs.dtype not in (torch.float32, torch.float64):
        llrs = llrs.to(torch.float64)
    if llrs.dim() != 2 or llrs.shape[1] != dg.N:
        raise ValueError("channel LLR length mismatch")
    fe = torch.as_tensor(np.ascontiguousarray(forced_edges), dtype=torch.int32).to(dev).contiguous()
    B, steps = llrs.shape[0], int(fe.shape[1]) if fe.dim() == 2 else 0
    if fe.dim() != 2 or fe.shape[0] != B:
        raise ValueError("forced_edges must be [B, steps]")
    if steps and (int(fe.min()) < 0 or int(fe.max()) >= dg.E):
        raise ValueError("forced edge out of range")
    cfg = ScheduleConfig(kind="rbp", kernel=kernel, precision=precision)
    sched = _sched(cfg, int(k_info or 0), llrs.dtype == torch.float64)
    L = _native.lib()
    sz = C.c_size_t()
    _native.check(L.ldpc_replay_workspace_size(dg.handle, C.byref(sched), B, C.byref(sz)),
                  "ldpc_replay_workspace_size")
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.stream(st):
        ws = torch.empty(max(sz.value, 256), dtype=torch.uint8, device=dev)
        trace = torch.empty((B, max(steps, 1)), dtype=torch.float64, device=dev)
        state = torch.empty((B, 2 * dg.E + 3 * dg.N), dtype=torch.float64, device=dev)
        counters = torch.empty((B, 8), dtype=torch.int64, device=dev)
    _native.check(L.ldpc_decode_replay(dg.handle, _ptr(llrs), B, C.byref(sched), _ptr(fe), steps, _ptr(trace),
                                       _ptr(state), _ptr(counters), _ptr(ws), ws.numel(),
                                       C.c_void_p(st.cuda_stream)), "ldpc_decode_replay")
    E, N = dg.E, dg.N
    return {"c2v_trace": trace[:, :steps], "c2v": state[:, :E], "pre_c2v": state[:, E:2 * E],
            "total": state[:, 2 * E:2 * E + N], "pre_total": state[:, 2 * E + N:2 * E + 2 * N],
            "ci": state[:, 2 * E + 2 * N:], "counters": counters, "_ws": ws}


def decode_batch_logged(code, llrs, config: ScheduleConfig, log_cap=1000, **kw):
    """decode_batch plus the propagated edge of each of the first `log_cap`
    updates per frame ([B, log_cap] int64, -1 past the end) and the committed
    C2V value (step_c2v, float64) -- debug and near-tie tracing against the
    CPU oracle's step log."""
    B = llrs.shape[0]
    dev = torch.device("cuda", torch.cuda.current_device())
    log = torch.full((B, log_cap, 2), -1, dtype=torch.int64, device=dev)
    L = _native.lib()
    _native.check(L.ldpc_set_step_log(_ptr(log), int(log_cap)), "ldpc_set_step_log")
    try:
        out = decode_batch(code, llrs, config, **kw)
    finally:
        L.ldpc_set_step_log(None, 0)
    out["step_log"] = log[:, :, 0]
    out["step_c2v"] = log[:, :, 1].view(torch.float64)
    return out
