"""The "compute-heavy end" of SURVEY.md §8(d) sweep-k: one 1920x1080 frame,
M = 1, a single window size k (21 or 31: beyond the TMA kernel's r_max = 6,
served by the v1 direct kernel, kmd_direct.cu), launched a few times for an
ncu capture of the FP32 pipe (scripts/gpu_final_r2.sh)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_05977_b200 import inputs as gen  # noqa: E402
from paper_2202_05977_b200 import kmd  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 21
dev = torch.device("cuda:0")
inp = gen.make_inputs(1, 1080, 1920, 1, with_blend=False, device=dev)
out = torch.empty((1, 3, 1080, 1920), device=dev)
for _ in range(6):
    kmd.decode_filter_fuse(inp.radiance, inp.importance, None, [k], out=out)
torch.cuda.synchronize()
print("k", k, kmd.last_kernel())
