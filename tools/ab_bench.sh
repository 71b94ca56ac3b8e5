#!/bin/bash
# A/B of tuning knobs on bench rows (development runs, under gpurun from the repo root):
#   TUNES="knob=0 knob=1" ROWS=row1,row2 bash tools/ab_bench.sh
# one line per (tuning, row) in gpurun_out/ab.txt: patterns/s (M) or Gq/s, checksum, roofline frac.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
ROWS=${ROWS:-c4_quadfm_approx1,c4_quadfm_approx1_bwt16x2,c5_reads_150bp_both_strands_approx1}
for t in $TUNES; do
  QR_TUNING=$t python bench.py --no-cpu --steps ${STEPS:-5} --warmup 3 --only $ROWS 2>>gpurun_out/ab.err | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for k,v in d['rows'].items():
    val = v.get('patterns_per_s', 0) / 1e6 if 'patterns_per_s' in v else v.get('gq_s')
    print('$t', k, round(val, 3) if val else val, v.get('checksum'), (v.get('roofline') or {}).get('frac'))
" >> gpurun_out/ab.txt
done
