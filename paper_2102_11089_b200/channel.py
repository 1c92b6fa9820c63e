"""BPSK over AWGN and channel LLRs (host side; the decoder's input generator).

Same conventions as the reference ``ldpc_ids.channel``
(/root/reference/pkg/src/ldpc_ids/channel.py):

* sigma = sqrt(1 / (2 R_tx 10^(Eb/N0/10))), R_tx = K / N_transmitted  (channel.py:35-40)
* LLR = clip(2y/sigma^2, +-30) at transmitted positions, 0 when punctured (channel.py:58-68)
* per-frame Philox(key=[master_seed, frame_index]) substreams           (channel.py:71-74)
* all-zero codeword, x = 1 - 2u, y = x + N(0, sigma^2)                   (channel.py:48-56, 77-86)

``llr_batch`` produces the [B, N] matrix the CUDA decoder consumes; rows are
bit-identical to ``generate_frame(code, cfg, start + b).channel_llrs``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

LLR_MAX = 30.0
RNG_NAME = "philox4x64"


@dataclass(frozen=True)
class ChannelConfig:
    ebn0_db: float
    sigma: float
    seed: int

    def __post_init__(self):
        if not self.sigma > 0:
            raise ValueError("sigma must be positive")


@dataclass
class Frame:
    u: np.ndarray
    y: np.ndarray
    channel_llrs: np.ndarray


def ebn0_to_sigma(ebn0_db, code):
    return float(np.sqrt(1.0 / (2.0 * code.rate_tx * 10.0 ** (ebn0_db / 10.0))))


def make_channel_config(ebn0_db, code, seed):
    return ChannelConfig(ebn0_db=ebn0_db, sigma=ebn0_to_sigma(ebn0_db, code), seed=seed)


def modulate(u):
    return 1.0 - 2.0 * np.asarray(u, dtype=np.float64)


def transmit(x, sigma, rng):
    return x + rng.normal(0.0, sigma, size=len(x))


def _transmitted_mask(code):
    mask = np.ones(code.h.n_cols, dtype=bool)
    mask[list(code.punctured)] = False
    return mask


def init_llrs(y, sigma, code):
    n = code.h.n_cols
    tx = _transmitted_mask(code)
    if len(y) != int(tx.sum()):
        raise ValueError(f"received vector length {len(y)} != transmitted count {int(tx.sum())}")
    llrs = np.zeros(n)
    llrs[tx] = np.clip(2.0 * np.asarray(y) / sigma ** 2, -LLR_MAX, LLR_MAX)
    return llrs


def frame_rng(master_seed, frame_index):
    key = np.array([master_seed, frame_index], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def generate_frame(code, config, frame_index):
    rng = frame_rng(config.seed, frame_index)
    n = code.h.n_cols
    u = np.zeros(n, dtype=np.int8)
    tx = _transmitted_mask(code)
    y = transmit(modulate(u[tx]), config.sigma, rng)
    return Frame(u=u, y=y, channel_llrs=init_llrs(y, config.sigma, code))


def llr_batch(code, ebn0_db, seed, start, count, dtype=np.float32):
    """[count, N] channel LLRs of frames start..start+count-1 (all-zero codeword).

    With dtype=float32 the rows are the fp32-rounded reference LLRs; the
    parity tests feed exactly these values (as float64) to the CPU oracle.
    """
    cfg = make_channel_config(ebn0_db, code, seed)
    n = code.h.n_cols
    tx = _transmitted_mask(code)
    n_tx = int(tx.sum())
    out = np.zeros((count, n), dtype=dtype)
    s2 = cfg.sigma ** 2
    for b in range(count):
        rng = frame_rng(seed, start + b)
        y = 1.0 + rng.normal(0.0, cfg.sigma, size=n_tx)
        out[b, tx] = np.clip(2.0 * y / s2, -LLR_MAX, LLR_MAX)
    return out


def llr_batch_device(code, ebn0_db, seed, start, count, dtype=None, device=None, stream=None):
    """[count, N] channel LLRs generated on the GPU (csrc/channel_gen.cu).

    Same channel model, LLR clip and puncturing as llr_batch and frames keyed
    by (seed, frame index), but a counter-based Philox4x32 + Box-Muller stream:
    statistically equivalent to the host generator, not bit-identical.  Needs
    prefix puncturing (apply_puncture).
    """
    import ctypes as C

    import torch

    from . import _native
    p = len(code.punctured)
    if tuple(code.punctured) != tuple(range(p)):
        raise ValueError("on-GPU generation supports prefix puncturing only")
    dtype = dtype or torch.float32
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    out = torch.empty((count, code.h.n_cols), dtype=dtype, device=device)
    st = stream if stream is not None else torch.cuda.current_stream(device)
    sigma = ebn0_to_sigma(ebn0_db, code)
    _native.check(_native.lib().ldpc_generate_awgn(code.h.n_cols, p, count, sigma, int(seed) & (2**64 - 1),
                                                   start, C.c_void_p(out.data_ptr()),
                                                   1 if dtype == torch.float64 else 0,
                                                   C.c_void_p(st.cuda_stream)),
                  "ldpc_generate_awgn")
    return out
