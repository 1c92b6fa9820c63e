"""B200-native informed-dynamic-schedule LDPC decoder.

Drop-in for the decode path of the reference package ``ldpc_ids``
(/root/reference/pkg/src/ldpc_ids): the same code-graph, channel and decoder
API names, with the schedule engine replaced by hand-written sm_100a CUDA
kernels behind a C ABI (include/ldpc_b200.h).
"""

from .channel import (ChannelConfig, Frame, ebn0_to_sigma, frame_rng, generate_frame,
                      init_llrs, llr_batch, make_channel_config, modulate, transmit)
from .codes import (BaseGraph, CodeError, CodeSpec, ParityCheckMatrix, TannerGraph,
                    apply_puncture, build_tanner, graph_stats, lift_base_graph,
                    make_random_regular_code, parse_base_graph, syndrome_ok)
from .kernels import Counters
from .schedules import (SCHEDULE_KINDS, DecodeResult, ScheduleConfig, decode, decode_batch,
                        select_vns)

__all__ = [n for n in dir() if not n.startswith("_")]
