# A/B of two library builds on one box for any command: the in-tree build (new) against
# gpurun_ab/old.so, alternating twice, programs compiled by each library (no program cache).
#   gpurun --timeout 1800 -- 'bash tools/ab_cmd.sh <tag> <command...>'
TAG=${1:-ab}; shift
mkdir -p gpurun_out
LIB=paper_2503_18616_b200/_native/libtissuesim_b200.so
cp $LIB gpurun_ab/new.so
export TS_PROGRAM_CACHE=0
for rep in 1 2; do
  for v in old new; do
    cp gpurun_ab/$v.so $LIB
    echo "== $v $rep"
    TAG=$v timeout 900 "$@" 2>&1 | tail -6
  done
done
cp gpurun_ab/new.so $LIB
