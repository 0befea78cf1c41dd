#!/bin/bash
# K2 A/B of library builds in build/variants/*.so against the bare memory pattern, same buffers,
# interleaved runs [tools/k2_vs_pattern.py with CANNIKIN_LIB].
set -u
mkdir -p gpurun_out
: > gpurun_out/k2_ab.jsonl
for rep in 1 2 3; do for lib in build/variants/*.so; do
  tag=$(basename $lib .so)
  CANNIKIN_LIB=$PWD/$lib timeout 300 python tools/k2_vs_pattern.py --sets synth --k2-grids 0 --pattern-grids 592 --tag $tag 2>/dev/null | grep '^{' >> gpurun_out/k2_ab.jsonl
done; done
