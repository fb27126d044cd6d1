"""Hashes of compiled programs over a matrix of scenes and layout options -- a refactor of the scene
compiler must leave every byte unchanged (development check; no GPU).

    TS_PROGRAM_CACHE=0 python tools/program_hashes.py > before.txt
"""
import dataclasses
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import build_slab_scene  # noqa: E402
from paper_2503_18616_b200 import scene as S  # noqa: E402
from paper_2503_18616_b200.mesh import default_scene_path, load_scene  # noqa: E402
from paper_2503_18616_b200 import _native as N  # noqa: E402


def dist_only(sc):
    mesh, rest, cfg = sc
    return (dataclasses.replace(mesh, tets=np.zeros((0, 4), np.int32)),
            dataclasses.replace(rest, rest_volume=np.zeros(0)), cfg)


reach = load_scene(default_scene_path())
slab = build_slab_scene(nx=6, ny=3, nz=3)
slab_att = build_slab_scene(nx=4, ny=2, nz=2, with_attachments=True)
cases = [
    ("reach f32", reach, {}),
    ("reach f32 384", reach, {"block_threads": 384}),
    ("reach f64", reach, {"precision": "fp64"}),
    ("reach f32 dist", dist_only(reach), {}),
    ("reach f32 noeg", reach, {"edge_gather": False}),
    ("reach f64 noeg", reach, {"precision": "fp64", "edge_gather": False}),
    ("reach f32 chunks", reach, {"max_chunk_slots": 1024}),
    ("reach f64 chunks", reach, {"precision": "fp64", "max_chunk_slots": 1024}),
    ("reach f32 nosched", reach, {"schedule_banks": False}),
    ("reach f32 noncompact", reach, {"compact": False}),
    ("slab f32", slab, {}),
    ("slab f64", slab, {"precision": "fp64"}),
    ("slab att f32", slab_att, {}),
    ("slab att f64", slab_att, {"precision": "fp64"}),
]
for name, sc, kw in cases:
    blob, info = S.compile_program(S.SceneArrays.from_loaded(*sc), **kw)
    print(f"{name:22s} {hashlib.sha256(blob.tobytes()).hexdigest()[:16]} {info['program_bytes']}", flush=True)
# cluster programs (one blob per part)
lib = N.load()
for name, sc, k, prec in (("reach K=2", reach, 2, "fp32"), ("reach K=4 f64", reach, 4, "fp64"),
                          ("slab K=2", slab, 2, "fp32")):
    blob, info = S.compile_program(S.SceneArrays.from_loaded(*sc), cluster_size=k, precision=prec)
    print(f"{name:22s} {hashlib.sha256(blob.tobytes()).hexdigest()[:16]} {info['program_bytes']}", flush=True)
