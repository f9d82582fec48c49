#!/bin/bash
# A/B of the systematic delivery pipelines (warp-subtile K2w/K3w vs the CTA-tile legacy K2/K3)
cd "$(dirname "$0")/.."
for m in default legacy; do
  echo "pipeline=$m"
  PFR_DV_PIPELINE=$m timeout 200 python scripts/fused_diag.py 2>&1
  PFR_DV_PIPELINE=$m DT=f64 LOGN=24 timeout 200 python scripts/fused_diag.py 2>&1
done
