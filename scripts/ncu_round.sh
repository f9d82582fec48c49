#!/bin/bash
# full ncu captures of the delivery kernels (systematic, 2^24 f32), Metropolis and rejection (2^20 f32)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
ncu --set full --clock-control none --import-source on -k "regex:k_dv_(reduce|expand|inplace)" -s 3 -c 3 \
    -o gpurun_out/${TAG:-r01}_deliver -f python scripts/profile_targets.py systematic 2 16777216 > gpurun_out/ncu_dv.txt 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_metropolis" -s 0 -c 1 \
    -o gpurun_out/${TAG:-r01}_metropolis -f python scripts/profile_targets.py metropolis 1 16777216 > gpurun_out/ncu_mh.txt 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_rej" -s 0 -c 2 \
    -o gpurun_out/${TAG:-r01}_rejection -f python scripts/profile_targets.py rejection 1 1048576 > gpurun_out/ncu_rj.txt 2>&1
echo done
