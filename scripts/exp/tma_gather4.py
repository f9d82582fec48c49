import ctypes, os, torch
here = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(here, "tma_gather4.so"))
lib.run.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
sink = torch.zeros(1, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
for log2n in (20, 24):
    buf = torch.rand(1 << log2n, device="cuda")
    for bps in (2, 4, 8):
        rows = 1 << 28
        st = torch.cuda.current_stream()
        rc = lib.run(buf.data_ptr(), log2n, rows, sink.data_ptr(), bps, st.cuda_stream); torch.cuda.synchronize()
        if rc: print("rc", rc); break
        ts = []
        for r in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); lib.run(buf.data_ptr(), log2n, rows, sink.data_ptr(), bps, st.cuda_stream); e1.record()
            torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ts.sort()
        per_iter = sms * bps * 4 * 32 * 2 * 4
        actual = per_iter * (rows // per_iter)
        print(f"2^{log2n} gather4 {bps} CTAs/SM: {actual / (ts[2] * 1e-3) / 1e9:6.1f} G rows/s", flush=True)
    del buf
