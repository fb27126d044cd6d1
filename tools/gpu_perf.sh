# Kernel iteration on one GPU: fp32/fp64 parity tests, a default bench line (no extras), the ncu
# launch list and one `ncu --set full` capture of the step kernel.
#   gpurun --timeout 1800 -- 'bash tools/gpu_perf.sh <tag>'
TAG=${1:-p}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fp32_parity.py tests/test_gpu_parity.py tests/test_gpu_env.py \
    tests/test_gpu_acceptance.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-extras > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "
import json
l=json.load(open('gpurun_out/bench_$TAG.json'))
print({k:l[k] for k in ('value','ms_per_step')}, l['e2e']['value'], {k:l['roofline'][k] for k in ('frac','kernel_ms','kernel')}, l['clocks'])
" || tail -5 gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-extras \
    > gpurun_out/launches_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 \
    -o gpurun_out/prof_step_$TAG -f python tools/profile_step.py > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu exit $?"
