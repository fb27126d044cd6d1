"""Single-env cluster timings (reach_1170 at K = 2, the 52,359-tet slab at K = 16) for A/B runs of
compiler / kernel variants (set the variant's environment before running)."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_mesh import gpu_rate  # noqa: E402
from paper_2503_18616_b200.mesh import default_scene_path, load_scene, make_slab_scene  # noqa: E402

d = tempfile.mkdtemp()
for name, scene, k in (("reach K=2", load_scene(default_scene_path()), 2),
                       ("reach K=4", load_scene(default_scene_path()), 4),
                       ("slab52k K=16", load_scene(make_slab_scene(d, tets=52359, name="s")), 16)):
    fps, ms, info = gpu_rate(scene, 1, 100, {"cluster_size": k})
    print(f"{os.environ.get('TAG', '')} {name}: {ms * 1e3:.1f} us/step", flush=True)
