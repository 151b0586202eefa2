#!/bin/bash
# A/B sweep of the timed-window kernels (C2 shape); one process per setting.
for mode in ${MODES:-lse hard}; do
  python scripts/time_c2.py $mode
  STLG_FAST=0 python scripts/time_c2.py $mode
  STLG_FAST=0 STLG_PIPE=0 python scripts/time_c2.py $mode
done
