# A/B of two builds of the library on one box: the in-tree build (B) against gpurun_ab/old.so (A),
# alternating, programs compiled by each library itself (no program cache).
#   gpurun --timeout 1800 -- 'bash tools/ab_lib.sh <tag> [bench args...]'
TAG=${1:-ab}; shift
mkdir -p gpurun_out
LIB=paper_2503_18616_b200/_native/libtissuesim_b200.so
cp $LIB gpurun_ab/new.so
export TS_PROGRAM_CACHE=0
for rep in 1 2; do
  for v in old new; do
    cp gpurun_ab/$v.so $LIB
    timeout 600 python bench.py --no-extras --no-cpu-baseline "$@" > gpurun_out/ab_${TAG}_${v}_$rep.json 2> gpurun_out/ab_${TAG}_${v}_$rep.err
    python -c "
import json; l=json.load(open('gpurun_out/ab_${TAG}_${v}_$rep.json'))
print('$v', $rep, round(l['value']), round(l['ms_per_step'], 5), round(l['roofline']['kernel_ms'], 5), l['roofline']['kernel'])" || tail -3 gpurun_out/ab_${TAG}_${v}_$rep.err
  done
done
cp gpurun_ab/new.so $LIB
