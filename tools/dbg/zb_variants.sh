#!/bin/bash
# Band-kernel occupancy variants: build the library with each define set (into
# build/variant.so, loaded through DCT16A_LIB; the product library is untouched) and
# time config 3 (path 0 = band kernel).  usage: zb_variants.sh "DEF1=a DEF2=b" ...
O=gpurun_out/zbv; mkdir -p $O
for v in "$@"; do
  python -c "
import sys; sys.path.insert(0, '.')
from paper_1606_05562_b200 import build
build.build(out='build/variant.so', defines=[d for d in '$v'.split() if d != 'base'])" > $O/build.log 2>&1 || { echo "build failed $v"; tail $O/build.log; continue; }
  echo "== $v"
  DCT16A_LIB=$PWD/build/variant.so timeout 300 python tools/time_zonal.py --paths 0 --r 16,32,64 --frames 600 2>&1 | grep "config 3"
done
