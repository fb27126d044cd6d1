# All bench configs + the mesh-scaling sweep on one GPU.   gpurun -- 'bash tools/gpu_configs.sh <tag>'
TAG=${1:-r01}
mkdir -p gpurun_out
for c in 3 1 2 5; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_c${c}_$TAG.json 2> gpurun_out/bench_c${c}_$TAG.err
  timeout 300 python bench.py --config $c --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c${c}_$TAG.json 2>> gpurun_out/bench_c${c}_$TAG.err
done
timeout 600 python bench.py --config 1 --cluster 4 --no-cpu-baseline > gpurun_out/bench_c1_k4_$TAG.json 2>> gpurun_out/bench_c1_$TAG.err
timeout 600 python bench.py --config 5 --envs 65536 --steps 20 --no-cpu-baseline > gpurun_out/bench_c5_65536_$TAG.json 2>> gpurun_out/bench_c5_$TAG.err
timeout 1200 python tools/bench_mesh.py --out gpurun_out/mesh_scaling_$TAG.json > gpurun_out/mesh_$TAG.log 2>&1
for f in gpurun_out/bench_*_$TAG.json; do echo "== $f"; cut -c1-400 $f; done
tail -3 gpurun_out/bench_c*_$TAG.err
cat gpurun_out/mesh_$TAG.log | cut -c1-600
