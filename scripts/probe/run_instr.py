"""Run the KMD_INSTR build of libkmd on a 1080p M=6 frame; print per-role wait cycles."""
import ctypes, os, shutil, sys
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import torch
from paper_2202_05977_b200 import kmd, inputs as gen
kmd.LIB_PATH = sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "libkmd_instr.so")
L = kmd.lib(build_if_missing=False)
L.kmd_debug_read_instr.argtypes = [ctypes.c_void_p, ctypes.c_int]
inp = gen.make_inputs(2, 1080, 1920, 6, device="cuda")
for _ in range(3):
    out = kmd.decode_filter_fuse(inp.radiance[:1], inp.importance[:1], inp.blend[:1], [3, 5, 7, 9, 11, 13])
torch.cuda.synchronize()
n = 160 * 16 * 16
buf = np.zeros(n, dtype=np.uint64)
L.kmd_debug_read_instr(buf.ctypes.data, n)
a = buf.reshape(160, 16, 16)[:148].astype(np.float64)
tags = ["rad_empty(TMA)", "in_empty(TMA)", "rad_full(F)", "v_empty(F)", "in_full(F)", "b_full(F)",
        "v_full(U)", "b_full(U)", "b_empty(TMA)", "fusebar1(U)", "fusebar2(U)", "epre_in_full(U)",
        "fuse_job(U)", "epilogue(U)"]
nw = int(os.environ.get("NWARPS", "11"))
for w in range(nw):
    tot = a[:, w, 15].mean()
    parts = ", ".join(f"{tags[t]}={a[:, w, t].mean() / tot:.0%}" for t in range(14) if a[:, w, t].mean() > 0)
    print(f"warp {w:2d}: total {tot / 1.9e3:.1f} us-equiv  waits: {parts}")
