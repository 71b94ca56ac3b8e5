# usage: bash /tmp/cmp.sh "variants" "rows" ; variant "def" = the in-tree library
cp paper_2602_04103_b200/lib/libqrank.so build/def.so
for v in $1; do
  if [ $v = def ]; then cp build/def.so paper_2602_04103_b200/lib/libqrank.so; else cp build/$v/libqrank.so paper_2602_04103_b200/lib/libqrank.so; fi
  python bench.py --no-cpu --steps 3 --warmup 3 --only $2 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for k,v in d['rows'].items(): print('$v', k, round(v.get('patterns_per_s',0)/1e6,2), v.get('checksum'), v.get('roofline',{}).get('frac'))
"
done
cp build/def.so paper_2602_04103_b200/lib/libqrank.so
