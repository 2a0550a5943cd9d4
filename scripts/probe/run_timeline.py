"""Per-CTA timeline of one 1080p M=6 launch (KMD_INSTR build): launch skew,
fill (first tile), per-tile pace and end spread, from %globaltimer."""
import ctypes, os, sys
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import torch
from paper_2202_05977_b200 import kmd, inputs as gen
kmd.LIB_PATH = sys.argv[1]
L = kmd.lib(build_if_missing=False)
H, W = int(os.environ.get("H", 1080)), int(os.environ.get("W", 1920))
inp = gen.make_inputs(1, H, W, 6, device="cuda")
for _ in range(5):
    out = kmd.decode_filter_fuse(inp.radiance, inp.importance, inp.blend, [3, 5, 7, 9, 11, 13])
torch.cuda.synchronize()
tl = np.zeros(160 * 16 * 2, dtype=np.uint64)
tt = np.zeros(160 * 16, dtype=np.uint64)
L.kmd_debug_read_timeline(tl.ctypes.data, tt.ctypes.data)
tl = tl.reshape(160, 16, 2)[:148].astype(np.float64)
tt = tt.reshape(160, 16)[:148].astype(np.float64)
t0 = tl[:, 0, 0].min()
b = tl[:, 0, 0] - t0
print(f"CTA begin skew: max {b.max()/1e3:.2f} us, median {np.median(b)/1e3:.2f}")
fw = int(os.environ.get("FUSE_W0", 5))
ends = tl[:, :12, 1] - t0
print(f"kernel span (first begin -> last end): {ends.max()/1e3:.2f} us")
for w, name in [(0, "TMA"), (1, "field0"), (fw, "fusion0")]:
    e = tl[:, w, 1] - t0
    print(f"{name:8s} end: min {e.min()/1e3:.2f} median {np.median(e)/1e3:.2f} max {e.max()/1e3:.2f} us")
nt = (tt > 0).sum(1)
print("tiles per CTA:", np.bincount(nt.astype(int)))
rel = (tt - t0) / 1e3
print("fusion tile-end times (us), percentiles over CTAs:")
for k in range(int(nt.max())):
    col = rel[nt > k, k]
    print(f"  tile {k}: p0 {col.min():.2f}  p50 {np.median(col):.2f}  p100 {col.max():.2f}")
last = np.array([rel[i, int(nt[i]) - 1] for i in range(148)])
order = np.argsort(-last)[:12]
print("slowest CTAs (cta: end us, first-tile end):", [(int(i), round(last[i], 2), round(rel[i, 0], 2)) for i in order])
q = np.arange(148) // 37
for g in range(4):
    print(f"  CTAs {g*37}-{g*37+36}: median end {np.median(last[q == g]):.2f} us")
print("per group (CTA // 37) median tile-end times:")
for g in range(4):
    print(f"  group {g}:", " ".join(f"{np.median(rel[q == g, k]):6.2f}" for k in range(int(nt.max()))))
d = np.diff(np.concatenate([np.zeros((148, 1)), rel], 1), axis=1)
print("per group median tile durations:")
for g in range(4):
    print(f"  group {g}:", " ".join(f"{np.median(d[q == g, k]):5.2f}" for k in range(int(nt.max()))))
