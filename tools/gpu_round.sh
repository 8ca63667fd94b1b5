#!/bin/bash
# One gpurun call: smoke, GPU tests, bench line (all legs), ncu launch list of the bench.
# Usage: tools/gpu_round.sh [tag]   (outputs under gpurun_out/<tag>/)
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --headline-only > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --headline-only > $O/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 $O/pytest_gpu.log
cat $O/bench.json | head -c 3000
