#!/bin/bash
# K1 output-path variants (DCT16A_FWD_STORE) under the current scheduler
for m in 3 4 5 6 7; do
  DCT16A_FWD_STORE=$m python tools/variants.py time --config 2 2>&1 | head -1 | sed "s/default/mode $m/"
done
