#!/bin/bash
# ncu_cases.sh TAG [CASE ...] -- run on the GPU box: one `ncu --set full`
# capture per tools/ncu_kernels.py case, exported right away to CSV (raw page
# for every launch; source page of the dominant kernel of C5) so that only
# small files come back in gpurun_out/ (the .ncu-rep files are removed).
#   tools/ncu_cases.sh r02b C5 C1 C3 C4 K7 io
#   python tools/ncu_summary.py --raw gpurun_out/ncu_r02b r02b
set -u
TAG=$1; shift
CASES=${*:-C5 C1 C3 C4 K7 io}
OUT=gpurun_out/ncu_$TAG
mkdir -p $OUT
for c in $CASES; do
  timeout 900 ncu --set full --clock-control none --import-source on -f -o $OUT/$c python tools/ncu_kernels.py $c \
    > $OUT/$c.log 2>&1
  echo "$c rc=$?"
  ncu -i $OUT/$c.ncu-rep --page raw --csv > $OUT/$c.raw.csv 2>> $OUT/$c.log
  if [ "$c" = "C5" ] || [ -n "${NCU_SOURCE:-}" ]; then
    ncu -i $OUT/$c.ncu-rep --page source --csv --print-source sass -k regex:k_roundtrip > $OUT/$c.source.csv 2>> $OUT/$c.log
  fi
  rm -f $OUT/$c.ncu-rep
done
du -sh $OUT
