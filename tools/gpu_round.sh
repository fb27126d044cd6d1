set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
TS_CHUNKS=0 TS_BLOCKS=0 python tools/tune.py > gpurun_out/tune.log 2>&1
python tools/train_ppo.py --max-updates 150 > gpurun_out/ppo.log 2>&1
python tools/train_ppo.py --max-updates 150 --window 100 > gpurun_out/ppo_w100.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/prof_step_f32 python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/tune.log; tail -4 gpurun_out/ppo.log; tail -2 gpurun_out/ppo_w100.log
