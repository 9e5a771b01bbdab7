#!/bin/bash
# ncu --set full of the first launch matching a kernel regex, exported on the GPU box as CSV pages
# (the .ncu-rep stays in /tmp: gpurun brings back <= 64 MiB):
#   tools/ncu_capture.sh <out_prefix> <kernel_regex> <skip> -- <command...>
# -> gpurun_out/<out_prefix>_raw.csv, <out_prefix>_sass.csv (per-instruction stall samples)
set -u
out=$1; rx=$2; skip=$3; shift 4
mkdir -p /tmp/rep gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:$rx" -s "$skip" -c 1 -o /tmp/rep/$out -f "$@" \
  > gpurun_out/${out}.log 2>&1
ncu -i /tmp/rep/$out.ncu-rep --page raw --csv > gpurun_out/${out}_raw.csv 2>>gpurun_out/${out}.log
ncu -i /tmp/rep/$out.ncu-rep --page source --csv --print-source sass > gpurun_out/${out}_sass.csv 2>>gpurun_out/${out}.log
ls -la gpurun_out/${out}*
