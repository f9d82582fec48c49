import ctypes, os, torch
here = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(here, "gather_paths.so"))
lib.run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
sink = torch.zeros(1, device="cuda")
for log2n in (20, 24, 28):
    buf = torch.rand(1 << log2n, device="cuda")
    for mode, name in ((0, "ldg.nc"), (1, "ldg.nc.no_allocate"), (2, "tex1Dfetch"), (3, "ldg.cg")):
        for gm in (4, 8):
            g = 1 << 29
            st = torch.cuda.current_stream()
            rc = lib.run(mode, buf.data_ptr(), log2n, g, sink.data_ptr(), gm, st.cuda_stream); torch.cuda.synchronize()
            ts = []
            for r in range(5):
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(); rc = lib.run(mode, buf.data_ptr(), log2n, g, sink.data_ptr(), gm, st.cuda_stream); e1.record()
                torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            ts.sort()
            sms = torch.cuda.get_device_properties(0).multi_processor_count
            actual = (sms * gm * 256) * 8 * (g // (sms * gm * 256 * 8))
            print(f"2^{log2n} {name:20s} grid x{gm}: {actual / (ts[2] * 1e-3) / 1e9:6.1f} G gathers/s (rc {rc})", flush=True)
    del buf
