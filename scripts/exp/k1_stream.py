import ctypes, os, subprocess, sys, torch
here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "k1_stream.so")
lib = ctypes.CDLL(so)
lib.run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
n = 1 << 24
w = torch.rand(n, device="cuda"); out = torch.zeros(1, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
mode = os.environ.get("FLUSH", "write")
st = torch.cuda.current_stream()
for which, gm in ((0, 0), (1, 0), (2, 2)):
    ts = []
    for r in range(12):
        if mode in ("write", "clean"):
            flush.zero_()
        if mode == "clean":
            clean.sum()
        torch.cuda._sleep(200000)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); rc = lib.run(which, w.data_ptr(), n, out.data_ptr(), gm, st.cuda_stream); e1.record()
        torch.cuda.synchronize(); assert rc == 0, rc
        if r >= 2: ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort(); print(f"flush {mode} kernel {which} grid_mult {gm}: median {ts[len(ts)//2]:.1f} us  -> {n*4/ts[len(ts)//2]/1e3:.0f} GB/s", flush=True)
