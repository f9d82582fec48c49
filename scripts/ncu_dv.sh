#!/bin/bash
# full ncu capture of the fused delivery kernels (systematic 2^24 f32), incl. the rare-path kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
ncu --set full --clock-control none --import-source on -k "regex:k_dv_" -s 4 -c 4 \
    -o gpurun_out/${TAG:-dv} -f python scripts/profile_targets.py systematic 2 ${NPOW:-16777216} > gpurun_out/ncu_dv.txt 2>&1
echo "ncu rc=$?"
