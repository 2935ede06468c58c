#!/bin/bash
# ncu --set full of one launch of a kernel in the bench workload (profile_run.py).
#   tools/ncu_kernel.sh <kernel-regex> <skip> <out-name> [profile_run args]
K=$1; SKIP=$2; OUT=$3; shift 3
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K -s $SKIP -c 1 -f -o gpurun_out/$OUT \
  python tools/profile_run.py --streams 64 "$@" > gpurun_out/$OUT.log 2>&1
tail -2 gpurun_out/$OUT.log
