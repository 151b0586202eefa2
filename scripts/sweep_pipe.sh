#!/bin/bash
# A/B of the timed F / G kernel families on the C2 workload (scripts/time_c2.py):
# register-blocked (default), the pipelined one-thread-per-block kernels
# (STLG_REG=0) and the non-pipelined ones (STLG_REG=0 STLG_PIPE=0).
for mode in lse hard soft; do
  python scripts/time_c2.py $mode
  STLG_REG=0 python scripts/time_c2.py $mode
  STLG_REG=0 STLG_PIPE=0 python scripts/time_c2.py $mode
done
