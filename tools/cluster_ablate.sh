# Single-env step time at K = 1 / 2 / 4 CTAs per env with parts of the step ablated (TS_ABLATE bits:
# 1 tets, 2 slot sums, 4 edge gather, 64 the whole substep loop) -- where the cluster time goes.
for ab in 0 64 5 7 1 4; do
  TS_ABLATE=$ab TAG="ablate=$ab" python - <<'PY'
import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
from bench_mesh import gpu_rate
from paper_2503_18616_b200.mesh import default_scene_path, load_scene
sc = load_scene(default_scene_path())
for k in (1, 2, 4):
    fps, ms, info = gpu_rate(sc, 1, 100, {"cluster_size": k} if k > 1 else None)
    print(os.environ["TAG"], f"K={k}", round(ms * 1e3, 1), "us", flush=True)
PY
done
