#!/bin/bash
# usage: prof_one.sh <name> <kernel-regex> <mode> [env...]  -> gpurun_out/<name>.ncu-rep
name=$1; kre=$2; mode=$3; shift 3
env "$@" python scripts/prof_c2.py $mode 3 > gpurun_out/plain_$name.log 2>&1 && \
env "$@" ncu --set full --import-source on --clock-control none -k regex:$kre -s 2 -c 1 -o gpurun_out/$name python scripts/prof_c2.py $mode 3 > gpurun_out/ncu_$name.log 2>&1
echo "$name rc=$?"
