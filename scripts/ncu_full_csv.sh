#!/bin/bash
# usage: ncu_full_csv.sh <name> <kernel-regex> <skip> <cmd...>
# One `ncu --set full` capture; the raw page is exported to gpurun_out/<name>.csv on the
# box (reports are ~30 MB each) and the report itself is kept only if KEEP_REP=1.
name=$1; kre=$2; skip=$3; shift 3
ncu --set full --import-source on --clock-control none -k regex:$kre -s $skip -c 1 -o gpurun_out/$name "$@" > gpurun_out/ncu_$name.log 2>&1
rc=$?
ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/$name.csv 2>/dev/null
ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>/dev/null
ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${name}_src.csv 2>/dev/null
[ "${KEEP_REP:-0}" = "1" ] || rm -f gpurun_out/$name.ncu-rep
echo "$name rc=$rc"
