# ncu of the config-2 edges kernel for the in-tree build and gpurun_ab/old.so (instruction and stall counts)
TAG=${1:-e}
LIB=paper_2503_18616_b200/_native/libtissuesim_b200.so
cp $LIB gpurun_ab/new.so
export TS_PROGRAM_CACHE=0 TS_DIST_ONLY=1 TS_ENVS=1024
for v in old new; do
  cp gpurun_ab/$v.so $LIB
  timeout 600 ncu --set full --clock-control none -k regex:edges_step -s 3 -c 1 -o gpurun_out/prof_edges_${TAG}_$v -f \
      python tools/profile_step.py > gpurun_out/ncu_edges_${TAG}_$v.log 2>&1
  echo "$v ncu exit $?"
done
cp gpurun_ab/new.so $LIB
