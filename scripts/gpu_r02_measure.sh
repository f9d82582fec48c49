#!/bin/bash
# Round-2 measurement pass: bench, ncu launch list of the bench step, ncu full
# captures of the delivery kernels (2^24 f32) and the bench's dominant kernels
# (rejection 2^20), sanitizer sweep of the new paths.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench.txt 2>&1; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-targets --no-cpu-baseline \
  > gpurun_out/r02_ncu_bench_stdout.txt 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_dv_(reduce|produce|resolve)" -s 3 -c 3 \
  -o gpurun_out/r02_deliver -f python scripts/profile_targets.py systematic 2 16777216 > /dev/null 2>&1; echo "ncu dv rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_rej" -s 0 -c 2 \
  -o gpurun_out/r02_rejection -f python scripts/profile_targets.py rejection 1 1048576 > /dev/null 2>&1; echo "ncu rej rc=$?"
if [ -n "$SANITIZE" ]; then
  for tool in memcheck racecheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_paths.py > gpurun_out/r02_sanitize_$tool.txt 2>&1
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_paths_large.py >> gpurun_out/r02_sanitize_$tool.txt 2>&1
    tail -2 gpurun_out/r02_sanitize_$tool.txt
  done
fi
