#!/bin/bash
# A/B timing of alternative builds: bash tools/ab.sh TAG ROUNDS dir1 dir2 ...
# ("-" = the in-tree library). Each round runs every variant once.
TAG=$1; ROUNDS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in $(seq 1 $ROUNDS); do
  for v in "$@"; do
    n=$(basename $v)
    if [ "$v" = "-" ]; then n=tree; lib=""; else lib=$(pwd)/$v/libcoopbatch_b200.so; fi
    CB_LIB_PATH=$lib timeout 600 python bench.py --no-cpu-baseline --no-evidence ${BENCH_ARGS:-} > $OUT/${n}_$r.json 2> $OUT/${n}_$r.err
  done
done
