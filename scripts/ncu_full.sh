#!/bin/bash
# full ncu capture of selected kernels: KREGEX, WHICH, N (log2)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_dv}" -s ${SKIP:-0} -c ${COUNT:-4} \
    -o gpurun_out/${OUT:-prof} -f python scripts/profile_targets.py ${WHICH:-systematic} 1 ${NPOW:-16777216} > gpurun_out/ncu_full_stdout.txt 2>&1
echo "ncu rc=$?"
