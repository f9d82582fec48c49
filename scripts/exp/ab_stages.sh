#!/bin/bash
# A/B: the fused delivery's stage times (scripts/time_stages.py) with prebuilt libpfr.so variants
cd "$(dirname "$0")/../.."
cp paper_1301_4019_b200/libpfr.so /tmp/libpfr_cur.so
for round in 1 2; do
for tag in "$@"; do
  cp scripts/exp/ab/libpfr_$tag.so paper_1301_4019_b200/libpfr.so
  echo "$tag: $(python scripts/time_stages.py 2>&1 | tr '\n' ' ')"
done
done
cp /tmp/libpfr_cur.so paper_1301_4019_b200/libpfr.so
