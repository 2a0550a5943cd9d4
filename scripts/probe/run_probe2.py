
import ctypes, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
if len(sys.argv) == 1:
    so = os.path.join(HERE, "probe2.so")
    cases = [(2,0,-12,1),(2,0,-30,1),(2,0,-35,1),(2,0,-36,1),(2,-8,-30,1),(2,8,-12,1),
             (4,0,0,1),(4,0,-12,1),(4,0,-6,1),(4,8,-12,1),(4,0,80,1),(4,180,80,1),(4,-8,0,1),(4,-4,-4,1)]
    for c in cases:
        r = subprocess.run([sys.executable, __file__, so] + [str(v) for v in c], capture_output=True, text=True, timeout=60)
        print("mode/cx/cy/l2", c, "|", " ".join(r.stdout.split())[-200:], flush=True)
    sys.exit(0)
import torch
L = ctypes.CDLL(sys.argv[1])
mode, cx, cy, l2 = map(int, sys.argv[2:6])
src = torch.arange(100 * 200, dtype=torch.float32, device="cuda").reshape(100, 200) + 1
out = torch.zeros(1, device="cuda")
torch.cuda.synchronize()
sys.stdout.flush()
rc = L.run_probe2(mode, cx, cy, l2, ctypes.c_void_p(src.data_ptr()), 200, 100, ctypes.c_void_p(out.data_ptr()))
if rc == 0 and mode != 4:
    x0, y0 = max(cx, 0), max(cy, 0)
    ref = src[y0:max(min(cy + 36, 100), 0), x0:max(min(cx + 64, 200), 0)].sum().item()
    print("sum", out.item(), "ref", ref, flush=True)
if rc == 0 and mode == 4:
    ones = (src == 1.0).sum().item()
    x0, y0 = max(cx, 0), max(cy, 0)
    exp = max(min(cy + 36, 100) - y0, 0) * max(min(cx + 64, 200) - x0, 0)
    print("ones", ones, "expected", exp, flush=True)
