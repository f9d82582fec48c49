#!/bin/bash
# Round-2 second measurement pass (after the rejection rework and the e2e
# schedule): bench, ncu launch list of the bench step, ncu full captures of
# the rejection kernels (f32 / f64, N=2^20: table + main kernel) and the
# delivery kernels (2^24 f32), sanitizers of the rejection paths.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02b_bench.txt 2>&1; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/r02b_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-targets --no-cpu-baseline \
  > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_rej" -s 0 -c 2 \
  -o gpurun_out/r02b_rejection_f32 -f python scripts/profile_targets.py rejection 1 1048576 > /dev/null 2>&1; echo "ncu rej32 rc=$?"
DT=f64 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_rej" -s 0 -c 2 \
  -o gpurun_out/r02b_rejection_f64 -f python scripts/profile_targets.py rejection 1 1048576 > /dev/null 2>&1; echo "ncu rej64 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_dv_(reduce|produce|resolve)" -s 3 -c 3 \
  -o gpurun_out/r02b_deliver -f python scripts/profile_targets.py systematic 2 16777216 > /dev/null 2>&1; echo "ncu dv rc=$?"
for tool in memcheck racecheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 10 python scripts/sanitize_rejection.py > gpurun_out/r02b_sanitize_$tool.txt 2>&1
  tail -1 gpurun_out/r02b_sanitize_$tool.txt
done
