#!/bin/bash
# A/B timing of environment settings: bash tools/ab_env.sh TAG ROUNDS "NAME=ENV ..." ...
# each variant is "label:VAR=value,VAR2=value" (label alone = defaults)
TAG=$1; ROUNDS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in $(seq 1 $ROUNDS); do
  for v in "$@"; do
    n=${v%%:*}; envs=${v#*:}; [ "$envs" = "$v" ] && envs=""
    env ${envs//,/ } timeout 600 python bench.py --no-cpu-baseline --no-evidence ${BENCH_ARGS:-} > $OUT/${n}_$r.json 2> $OUT/${n}_$r.err
  done
done
