#!/bin/bash
# Warp-kernel (config 4) build variants: build the library with each define
# set into build/variant.so (loaded through DCT16A_LIB; the product library is untouched)
# and time 300 config-4 frames at Δ = 16.  usage: cw_variants.sh "DEF=a DEF=b" ...
O=gpurun_out/cwv; mkdir -p $O
for v in "$@"; do
  python -c "
import sys; sys.path.insert(0, '.')
from paper_1606_05562_b200 import build
build.build(out='build/variant.so', defines=[d for d in '$v'.split() if d != 'base'])" > $O/build.log 2>&1 || { echo "build failed $v"; tail $O/build.log; continue; }
  echo "== $v"
  DCT16A_LIB=$PWD/build/variant.so timeout 300 python tools/time_cfg4.py --frames 300 --steps 16 --paths 2,2 2>&1 | tail -1 | cut -c1-200
done
