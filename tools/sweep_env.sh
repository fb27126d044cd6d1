# Default bench line under compiler environment knobs (fresh programs each time).
#   gpurun -- 'bash tools/sweep_env.sh "TS_PIN_COPIES=2" "TS_PIN_COPIES=1" ...'
for kv in "" "$@"; do
  env $kv TS_PROGRAM_CACHE=0 timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 100 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.readline()); print('[$kv]', round(l['value']), round(l['ms_per_step'],5), round(l['roofline']['kernel_ms'],5))" || echo "[$kv] failed"
done
