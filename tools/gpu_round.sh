set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
TS_CHUNKS=0,6000,4200,3000 python tools/tune.py > gpurun_out/tune.log 2>&1
tail -4 gpurun_out/pytest_gpu.log; cat gpurun_out/tune.log
