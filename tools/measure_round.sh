set -u
T=${1:-r02f}
python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/${T}_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke=$?"
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_reference_arm.json 2>/dev/null; echo "ref=$?"
python tools/shard_probe.py > gpurun_out/${T}_shard_probe.json 2>gpurun_out/${T}_shard_probe.err; echo "shard=$?"
python tools/shard_probe.py --c5 > gpurun_out/${T}_shard_probe_c5.json 2>>gpurun_out/${T}_shard_probe.err; echo "shard_c5=$?"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_smoke.py > gpurun_out/${T}_san_$tool.log 2>&1; echo "$tool=$?"; tail -3 gpurun_out/${T}_san_$tool.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-configs --probe-steps 2 > /dev/null 2>&1; echo "launches=$?"
bash tools/ncu_cases.sh $T C5 C1 C3 C4 K7 io
