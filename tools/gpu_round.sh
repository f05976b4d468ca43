#!/bin/bash
# One GPU-box pass: parity tests, bench line, launch list, ncu captures.
# usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
KR="regex:batch_begin|frontier|labor|post_kernel|relabel|gather|ns_|extract|fused|vtab"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" --csv \
  --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-evidence > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather -s 3 -c 1 \
  -o $OUT/gather_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-evidence > $OUT/ncu_gather.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:labor_mark -s 8 -c 1 \
  -o $OUT/labor_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-evidence > $OUT/ncu_labor.log 2>&1
echo done > $OUT/DONE
