#!/bin/bash
# Round-2 closing pass: build, full GPU suite, smoke, bench, launch list,
# ncu captures of the dominant kernels, sanitizers of the reworked paths.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02c_pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02c_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02c_bench.txt 2>&1; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/r02c_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-targets --no-cpu-baseline \
  > /dev/null 2>&1; echo "ncu launches rc=$?"
for d in f32 f64; do
  DT=$d timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_rej" -s 0 -c 2 \
    -o gpurun_out/r02c_rejection_$d -f python scripts/profile_targets.py rejection 1 1048576 > /dev/null 2>&1; echo "ncu rej $d rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_mn_|k_sc_" -s 0 -c 6 \
  -o gpurun_out/r02c_multinomial -f python scripts/profile_targets.py multinomial 1 1048576 > /dev/null 2>&1; echo "ncu mn rc=$?"
cat > /tmp/san_mn.py <<'PY'
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_1301_4019_b200 as pf
for n in (1, 7, 1023, 1025, 4097, 70001, (1 << 20) + 3):
    for dt in (np.float32, np.float64):
        w = np.exp(np.random.default_rng(n).normal(0, 1, n)).astype(dt)
        w[::7] = 0
        if not w.any(): w[0] = 1
        a = pf.multinomial_ancestors(w, pf.RngStream(3))
        assert int(a.min()) >= 0 and int(a.max()) < n
print("sanitize multinomial ok")
PY
for tool in memcheck racecheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 10 python /tmp/san_mn.py > gpurun_out/r02c_sanitize_mn_$tool.txt 2>&1
  tail -1 gpurun_out/r02c_sanitize_mn_$tool.txt
  timeout 600 compute-sanitizer --tool $tool --print-limit 10 python scripts/sanitize_rejection.py > gpurun_out/r02c_sanitize_rej_$tool.txt 2>&1
  tail -1 gpurun_out/r02c_sanitize_rej_$tool.txt
done
