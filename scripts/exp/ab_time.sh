#!/bin/bash
# A/B: time one op with two prebuilt libpfr.so variants (scripts/exp/ab/libpfr_<tag>.so)
cd "$(dirname "$0")/../.."
cp paper_1301_4019_b200/libpfr.so /tmp/libpfr_cur.so
for round in 1 2; do
for tag in "$@"; do
  cp scripts/exp/ab/libpfr_$tag.so paper_1301_4019_b200/libpfr.so
  for dt in f32 f64; do echo "$tag rejection $dt: $(python scripts/time_ops.py rejection 20 $dt 2>&1 | tail -1)"; done
  echo "$tag metropolis f32: $(python scripts/time_ops.py metropolis 20 f32 2>&1 | tail -1)"
done
done
cp /tmp/libpfr_cur.so paper_1301_4019_b200/libpfr.so
