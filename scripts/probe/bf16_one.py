import sys, torch
sys.path.insert(0, '.')
from paper_2202_05977_b200 import inputs as gen, kmd
sizes = [int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "3,5,7,9,11,13").split(",")]
H, W = 96, int(sys.argv[2]) if len(sys.argv) > 2 else 160
inp = gen.make_inputs(1, H, W, len(sizes), seed=301, device="cuda")
i16 = inp.importance.to(torch.bfloat16); b16 = None if inp.blend is None else inp.blend.to(torch.bfloat16)
o = kmd.decode_filter_fuse(inp.radiance, i16, b16, sizes)
torch.cuda.synchronize()
print("ok", kmd.last_kernel(), float(o.abs().max()))
