#!/bin/bash
# ab_vs_head.sh -- on the GPU box: the config sub-keys and the C5 headline of
# the working tree's build against a HEAD build, two rounds, plus the codec /
# pipeline GPU tests.  Prepare here first:
#   git stash && python tools/build_variant.py head && git stash pop
#   python -c "import __graft_entry__ as g; g.build()"
#   gpurun -- 'bash tools/ab_vs_head.sh'
python -m pytest tests -m gpu -x -q -k "codec or pipeline or fullsize or sharded" 2>&1 | tail -1
for r in 1 2; do
for v in new head; do
  if [ $v = head ]; then export OPTB_CUDA_LIB=_ab/head.so; else unset OPTB_CUDA_LIB; fi
  python tools/cfg_ab.py C1_exact64 C3 C4_exact128 C2_sbs 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', d['case'], d['value'], d['roundtrip_us'] or d['ms_per_step'], d['hbm_frac'], d['encode_us'], d['encode_frac'], d['decode_frac'], d['check'])"
  python bench.py --no-configs --no-cpu-baseline --e2e-steps 0 --steps 50 2>/dev/null | python3 -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v C5', d['value'], d['ms_per_step'], d['roofline']['frac'], d['check']['ok'])"
done
done
