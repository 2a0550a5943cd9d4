import ctypes, os, sys, torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "tma_stream.so"))
L.run_stream.restype = ctypes.c_float
W, H, P = 1920, 1080, 24   # 24 planes ~ 4 frames x 6 maps (199 MB)
src = torch.randn(P, H, W, device="cuda")
sink = torch.zeros(1, device="cuda")
for rows in (36, 72):
    for ns in (2, 4, 8, 16):
        for cps in (1, 2):
            smem = ns * rows * 68 * 4
            if smem * cps > 220 * 1024: continue
            ms = L.run_stream(ctypes.c_void_p(src.data_ptr()), W, H, P, ns, rows, cps, ctypes.c_void_p(sink.data_ptr()))
            tiles = ((W + 51) // 52) * ((H + rows - 13) // (rows - 12)) * P
            box_bytes = tiles * rows * 68 * 4
            print(f"rows={rows} ns={ns} ctas/SM={cps} inflight/SM={ns*rows*68*4*cps/1024:.0f}KB: {ms*1000:.1f} us, "
                  f"payload {box_bytes/ms/1e6:.0f} GB/s, unique {P*H*W*4/ms/1e6:.0f} GB/s", flush=True)
