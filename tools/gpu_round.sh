# One GPU round: tests, smoke, bench line, reference arm, ncu launch list, one full ncu capture of the
# step kernel, compute-sanitizer memcheck / racecheck on the production (and latency) programs.
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh <tag>'
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi_$TAG.txt 2>&1
lscpu > gpurun_out/lscpu_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-extras \
    > gpurun_out/launches_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 \
    -o gpurun_out/prof_step_$TAG -f python tools/profile_step.py > gpurun_out/ncu_full_$TAG.log 2>&1
for tool in memcheck racecheck; do
  TS_ENVS=160 TS_STEPS=2 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_step.py \
      > gpurun_out/sanitize_${tool}_$TAG.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${tool}_$TAG.txt
done
tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log; cat gpurun_out/bench_ref_$TAG.json
tail -3 gpurun_out/sanitize_memcheck_$TAG.txt gpurun_out/sanitize_racecheck_$TAG.txt
