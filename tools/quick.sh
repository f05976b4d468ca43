#!/bin/bash
# Iteration loop on the GPU box: parity tests, then 2 short bench lines.
# usage: bash tools/quick.sh TAG [pytest-args]
TAG=${1:-q}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q "$@" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-evidence > $OUT/bench$i.json 2> $OUT/bench$i.err; done
