set -u
OUT=gpurun_out/ncu_ll
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(decode_vec|encode_bulk|encode_vec)" -c 4 -f -o $OUT/ll python tools/ncu_kernels.py C3L > $OUT/ll.log 2>&1
echo rc=$?
ncu -i $OUT/ll.ncu-rep --page raw --csv > $OUT/ll.raw.csv 2>> $OUT/ll.log
ncu -i $OUT/ll.ncu-rep --page source --csv --print-source sass > $OUT/ll.source.csv 2>> $OUT/ll.log
ls -la $OUT
rm -f $OUT/ll.ncu-rep
