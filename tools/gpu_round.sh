set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1
python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
python tools/train_ppo.py --max-updates 120 > gpurun_out/ppo.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -c 2500 gpurun_out/bench.log; tail -c 1500 gpurun_out/bench_ref.log; tail -25 gpurun_out/ppo.log
