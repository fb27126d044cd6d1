# Sweep the phase-1 work-split weight of a tet batch vs an edge round (compiler TS_SPLIT_CT), fresh
# programs each time; prints the fast kernel's time per step.
#   gpurun --timeout 1200 -- 'bash tools/sweep_ct.sh 3 4 5 6'
for ct in "$@"; do
  TS_SPLIT_CT=$ct TS_PROGRAM_CACHE=0 timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 30 \
      > gpurun_out/sweep_ct_$ct.json 2>/dev/null
  python -c "
import json; l=json.load(open('gpurun_out/sweep_ct_$ct.json'))
print('CT=$ct', round(l['roofline']['kernel_ms'],4), round(l['ms_per_step'],4), round(l['value']))" || echo "CT=$ct failed"
done
