import ctypes, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
if len(sys.argv) == 1:
    for build in ["static", "shared"]:
        so = os.path.join(HERE, f"probe_{build}.so")
        for v in (0, 1, 4, 5):
            r = subprocess.run([sys.executable, __file__, so, str(v)], capture_output=True, text=True, timeout=60)
            print(build, v, r.returncode, r.stdout.strip()[-400:], flush=True)
    sys.exit(0)
import torch
L = ctypes.CDLL(sys.argv[1])
src = torch.arange(100 * 200, dtype=torch.float32, device="cuda").reshape(100, 200)
out = torch.zeros(1, device="cuda")
sys.stdout.flush()
rc = L.run_probe(int(sys.argv[2]), ctypes.c_void_p(src.data_ptr()), 200, 100, ctypes.c_void_p(out.data_ptr()))
print("rc", rc, flush=True)
torch.cuda.synchronize()
ref = src[:30, :58].sum().item()
print("rc", rc, "sum", out.item(), "ref", ref)
