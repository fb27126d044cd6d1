# Quick GPU iteration: selected tests, smoke, default bench line.
#   gpurun --timeout 1500 -- 'bash tools/gpu_quick.sh <tag> [pytest selectors...]'
TAG=${1:-q}; shift
mkdir -p gpurun_out
if [ $# -gt 0 ]; then
  timeout 900 python -m pytest "$@" -m gpu -q -x -s -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
  tail -15 gpurun_out/pytest_$TAG.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
tail -4 gpurun_out/smoke_$TAG.log
T0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench wall $(( $(date +%s) - T0 )) s"
tail -3 gpurun_out/bench_$TAG.err
python -c "
import json,sys
l=json.load(open('gpurun_out/bench_$TAG.json'))
print({k:l[k] for k in ('value','ms_per_step','gpu_launches')}, l['e2e'], {k:l['roofline'][k] for k in ('frac','kernel_ms')})
for k,v in l.get('extras',{}).items():
    if isinstance(v,dict) and 'value' in v: print(k, round(v['value']), round(v['ms_per_step'],4), v['roofline']['frac'], v['roofline']['kernel'], v.get('cpu_baseline',{}).get('value'))
    elif isinstance(v,dict): print(k, {kk:v[kk] for kk in ('reward_crossed_at_env_steps','reward_crossed_wall_s','wall_s','updates','eval_greedy_500_episodes') if kk in v})
    else: print(k, v)
"
