#!/bin/bash
# Round-end evidence in one gpurun call: smoke, every GPU test, the bench line
# (all legs), the reference arm, the ncu launch list of the bench, and ncu
# --set full captures of the dominant kernels (forward on config 2, band
# kernel on config 3, warp kernel on config 4).
TAG=${1:-r02_final}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/reference.json 2> $O/reference.err; echo "ref rc=$?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --headline-only > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --headline-only > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fwd_kernel -s 1 -c 1 -o $O/fwd_full \
   python tools/prof_fwd.py > $O/ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:zband -c 1 -o $O/zb_full \
   python tools/prof_codec.py --config 3 --frames 100 --launches 2 > $O/ncu_zb.log 2>&1; echo "ncu zb rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:codec_warp -c 1 -o $O/cw_full \
   python tools/prof_codec.py --config 4 --frames 50 --launches 2 > $O/ncu_cw.log 2>&1; echo "ncu cw rc=$?"
tail -3 $O/pytest_gpu.log
head -c 1500 $O/bench.json
