# Time the default bench line with each library variant gpurun_ab/var_*.so (twice, interleaved),
# programs compiled by each library (no program cache).  Restores the in-tree build afterwards.
#   gpurun --timeout 2400 -- 'bash tools/ab_multi.sh [bench args...]'
LIB=paper_2503_18616_b200/_native/libtissuesim_b200.so
cp $LIB gpurun_ab/intree.so
export TS_PROGRAM_CACHE=0
for rep in 1 2; do
  for f in gpurun_ab/var_*.so; do
    cp $f $LIB
    v=$(basename $f .so)
    timeout 600 python bench.py --no-extras --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.readline()); print('$v', $rep, round(l['value']), round(l['ms_per_step'],5), round(l['roofline']['kernel_ms'],5))" || echo "$v failed"
  done
done
cp gpurun_ab/intree.so $LIB
