#!/bin/bash
# One GPU round trip: build, GPU parity tests, smoke, short bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests/ -m gpu -q --timeout 600 -rf --tb=short ${PYTEST_ARGS} > gpurun_out/gpu_tests.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.txt
tail -5 gpurun_out/gpu_tests.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
tail -2 gpurun_out/smoke.txt
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py --steps ${STEPS:-3} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/bench.txt
  tail -c 3000 gpurun_out/bench.txt
fi
if [ -n "$SANITIZE" ]; then
  for tool in memcheck racecheck synccheck; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_paths.py > gpurun_out/sanitize_$tool.txt 2>&1
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_paths_large.py >> gpurun_out/sanitize_$tool.txt 2>&1
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_paths_modes.py >> gpurun_out/sanitize_$tool.txt 2>&1
    tail -1 gpurun_out/sanitize_$tool.txt
  done
fi
