#!/bin/bash
# A/B of compile-time variants on bench rows (development runs, under gpurun from the repo root):
#   VARIANTS="def v3:-DQR_AX1_PATH_MINB=3" ROWS=row1,row2 bash tools/ab_builds.sh
# "def" is the in-tree build; name:flags builds build/<name>/libqrank.so with QR_EXTRA=flags.
# One line per (variant, row) in gpurun_out/ab.txt.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
make -s all > gpurun_out/make.log 2>&1
LIB=paper_2602_04103_b200/lib/libqrank.so
cp $LIB build/def.so
for v in $VARIANTS; do
  name=${v%%:*}; flags=${v#*:}
  if [ "$name" != def ]; then
    rm -rf build/$name; mkdir -p build/$name
    make -s -B BUILD=build/$name QR_EXTRA="$flags" $LIB >> gpurun_out/make.log 2>&1 && cp $LIB build/$name/libqrank.so
  fi
done
for rep in 1 2; do
  for v in $VARIANTS; do
    name=${v%%:*}
    if [ "$name" = def ]; then cp build/def.so $LIB; else cp build/$name/libqrank.so $LIB; fi
    python bench.py --no-cpu --steps ${STEPS:-5} --warmup 3 --only $ROWS 2>>gpurun_out/ab.err | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for k,v in d['rows'].items():
    val = v.get('patterns_per_s', 0) / 1e6 if 'patterns_per_s' in v else v.get('gq_s')
    print('$name', k, round(val, 3) if val else val, v.get('checksum'), (v.get('roofline') or {}).get('frac'))
" >> gpurun_out/ab.txt
  done
done
cp build/def.so $LIB
