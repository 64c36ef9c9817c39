#!/bin/bash
# ncu_case_source.sh TAG CASE KERNEL_REGEX COUNT -- run on the GPU box: one
# `ncu --set full` capture of tools/ncu_kernels.py CASE restricted to the
# kernels matching KERNEL_REGEX (first COUNT launches), exported to CSV (raw
# page + SASS source page) under gpurun_out/ncu_TAG/; for
# tools/ncu_source_lines.py.
set -u
TAG=$1; CASE=$2; KRE=$3; CNT=${4:-2}
OUT=gpurun_out/ncu_$TAG
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c $CNT -f -o $OUT/$CASE \
  python tools/ncu_kernels.py $CASE > $OUT/$CASE.log 2>&1
echo "rc=$?"
ncu -i $OUT/$CASE.ncu-rep --page raw --csv > $OUT/$CASE.raw.csv 2>> $OUT/$CASE.log
ncu -i $OUT/$CASE.ncu-rep --page source --csv --print-source sass > $OUT/$CASE.source.csv 2>> $OUT/$CASE.log
rm -f $OUT/$CASE.ncu-rep
ls -la $OUT
