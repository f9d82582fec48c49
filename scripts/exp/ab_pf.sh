#!/bin/bash
# A/B: the batched filter (512 x 2^16 x 100) with prebuilt libpfr.so variants
cd "$(dirname "$0")/../.."
cp paper_1301_4019_b200/libpfr.so /tmp/libpfr_cur.so
for round in 1 2; do
for tag in "$@"; do
  cp scripts/exp/ab/libpfr_$tag.so paper_1301_4019_b200/libpfr.so
  echo "$tag: $(python scripts/pf_time.py 512 100 2>&1 | tail -1)"
done
done
cp /tmp/libpfr_cur.so paper_1301_4019_b200/libpfr.so
