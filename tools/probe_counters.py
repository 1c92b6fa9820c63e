import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import pyoracle
from paper_2102_11089_b200.channel import llr_batch
from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch, results_to_numpy
from tests.util import load_code
spec, g = load_code("C1")
llr = llr_batch(spec, 2.0, 0, 0, 128)
cfg = ScheduleConfig(kind="me_cirbp", i_max=3, n_p=4)
got = results_to_numpy(decode_batch(spec, torch.from_numpy(llr).cuda(), cfg), "me_cirbp", 3)
ref = pyoracle.decode_batch(g, llr.astype(np.float64), "me_cirbp", i_max=3, k_info=spec.k_info, n_p=4)
bad = np.flatnonzero(~(got["counters"] == ref["counters"]).all(1))
for b in bad:
    print(b, got["counters"][b].tolist(), ref["counters"][b].tolist(), got["prop"][b], ref["prop"][b])
