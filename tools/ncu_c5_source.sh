#!/bin/bash
# ncu_c5_source.sh TAG -- run on the GPU box: one `ncu --set full` capture of
# the C5 pipeline step's round-trip kernel with source counters, exported to
# CSV (raw + SASS source page) under gpurun_out/ncu_TAG/.
set -u
TAG=$1
OUT=gpurun_out/ncu_$TAG
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_roundtrip -c 1 -f -o $OUT/c5 \
  python tools/ncu_kernels.py C5 > $OUT/c5.log 2>&1
echo "rc=$?"
ncu -i $OUT/c5.ncu-rep --page raw --csv > $OUT/c5.raw.csv 2>> $OUT/c5.log
ncu -i $OUT/c5.ncu-rep --page source --csv --print-source sass > $OUT/c5.source.csv 2>> $OUT/c5.log
rm -f $OUT/c5.ncu-rep
ls -la $OUT
