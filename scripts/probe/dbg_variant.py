"""Run one small case on a given libkmd build and report where it differs from the oracle."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_05977_b200 import kmd, inputs as gen
import oracle
kmd.LIB_PATH = sys.argv[1]
for (H, W, sizes) in [(64, 64, [5]), (54, 104, [3, 5, 7, 9, 11, 13]), (27, 52, [3])]:
    inp = gen.make_inputs(1, H, W, len(sizes), seed=1)
    try:
        out = kmd.decode_filter_fuse(inp.radiance.cuda(), inp.importance.cuda(),
                                     None if inp.blend is None else inp.blend.cuda(), sizes)
        torch.cuda.synchronize()
    except Exception as e:
        print(H, W, sizes, "ERROR", e); continue
    ref = oracle.decode_filter_fuse(inp.radiance.numpy(), inp.importance.numpy(),
                                    None if inp.blend is None else inp.blend.numpy(), sizes)
    got = out.cpu().numpy()
    rel = np.abs(got - ref) / np.abs(ref)
    bad = np.argwhere(rel > 1e-5)
    print(H, W, sizes, kmd.last_kernel(), "max rel", np.nanmax(rel), "bad", len(bad))
    if len(bad):
        ys = sorted(set(int(b[2]) for b in bad)); xs = sorted(set(int(b[3]) for b in bad))
        print("  rows", ys[:30], "cols", xs[:60])
