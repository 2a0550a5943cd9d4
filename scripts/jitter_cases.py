"""Outputs of the pipelined kernels on fixed inputs, saved for a bitwise
comparison across runs (tests/test_gpu_checked.py): run with KMD_LIB = the
checked library and KMD_DEBUG = a scheduling-jitter seed (0 = none).

    python scripts/jitter_cases.py OUT_DIR
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2202_05977_b200 import inputs as gen  # noqa: E402
from paper_2202_05977_b200 import kmd  # noqa: E402

out_dir = sys.argv[1]
os.makedirs(out_dir, exist_ok=True)
dev = torch.device("cuda:0")
PAPER = list(gen.PAPER_SIZES)

# 1080p, M = 6: 10 tiles per CTA, every ring wraps many times
inp = gen.make_inputs(1, 1080, 1920, 6, seed=91)
r, i, b = inp.radiance.to(dev), inp.importance.to(dev), inp.blend.to(dev)
o = kmd.decode_filter_fuse(r, i, b, PAPER)
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
o = kmd.decode_filter_fuse(r, i, b, PAPER)
t1.record()
torch.cuda.synchronize()
print(f"1080p M=6 launch: {t0.elapsed_time(t1) * 1e3:.1f} us (jitter seed {os.environ.get('KMD_DEBUG', '0')})")
assert kmd.last_kernel() == "v3-tma-M6", kmd.last_kernel()
np.save(os.path.join(out_dir, "m6.npy"), o.cpu().numpy())

# runtime-M kernel and the border variant on a batch of 3 small frames
inp = gen.make_inputs(3, 200, 312, 3, seed=92)
o = kmd.decode_filter_fuse(inp.radiance.to(dev), inp.importance.to(dev), inp.blend.to(dev), [3, 7, 13])
torch.cuda.synchronize()
np.save(os.path.join(out_dir, "m3.npy"), o.cpu().numpy())

# "Ours MR" (three level launches with the Eq. 7 epilogue)
mi = gen.make_mr_inputs(1, 540, 960)
o = kmd.mr_decode_filter_fuse(mi.radiance.to(dev), [t.to(dev) for t in mi.importance],
                              [t.to(dev) for t in mi.blend], [t.to(dev) for t in mi.alpha],
                              [list(s) for s in gen.MR_SIZES])
torch.cuda.synchronize()
assert kmd.last_kernel() == "v3-tma28-mr-cmb", kmd.last_kernel()
np.save(os.path.join(out_dir, "mr.npy"), o.cpu().numpy())
print("jitter cases done")
