#!/bin/bash
# A/B of sampler variants on the bench workload (per-period timing).
# usage: tools/ab.sh "VAR=val ..." "VAR=val ..."   (each arg: env settings of one variant)
for v in "$@"; do
  echo "== $v"
  env $v python tools/period_timing.py --periods 8 2>&1 | tail -n 3
done
