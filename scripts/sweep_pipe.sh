#!/bin/bash
# A/B sweep of the pipelined timed-window kernels (C2 shape); one process per setting.
for mode in ${MODES:-lse hard}; do
  python scripts/time_c2.py $mode
  STLG_PIPE_SKIP=1 python scripts/time_c2.py $mode
  STLG_PIPE_SKIP=2 python scripts/time_c2.py $mode
  STLG_PIPE_NB=48 python scripts/time_c2.py $mode
  STLG_PIPE_NB=40 python scripts/time_c2.py $mode
  STLG_PIPE=0 python scripts/time_c2.py $mode
done
