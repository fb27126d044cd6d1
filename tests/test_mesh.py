"""Scene ingest: bit-exact topology and rest data vs the reference (golden), parser errors, fixtures.

Mirrors pkg/tests/test_mesh.py (topology counts, face oracle, slab face count,
outward winding, volumes, parse errors) and pins every index array against
tests/golden/topology.npz produced by the reference.
"""

import collections
import filecmp
import os

import numpy as np
import pytest

from conftest import build_slab_scene, golden
from paper_2503_18616_b200.errors import ParseError, ValidationError
from paper_2503_18616_b200.mesh import (
    SceneConfig, build_mesh, compute_rest_state, derive_topology, fix_orientation, load_scene, make_slab,
    make_slab_scene, parse_mesh_text, parse_scene_text, signed_volumes, write_mesh, write_scene,
)


def surface_faces_oracle(tets):
    counts = collections.Counter()
    for a, b, c, d in np.asarray(tets).tolist():
        for tri in ((a, b, c), (a, b, d), (a, c, d), (b, c, d)):
            counts[tuple(sorted(tri))] += 1
    return {tri for tri, n in counts.items() if n == 1}


class TestGoldenTopology:
    def test_reach_1170_bit_exact(self, reach_scene):
        mesh, rest, cfg = reach_scene
        g = golden("topology.npz")
        for key in ("positions_rest", "tets", "edges", "surface_faces", "pinned", "vertex_mass"):
            a = getattr(mesh, key)
            assert a.dtype == g[key].dtype, key
            assert np.array_equal(a, g[key]), key
        for key in ("rest_length", "rest_volume", "inverse_mass"):
            assert np.array_equal(getattr(rest, key), g[key]), key
        assert (mesh.vertex_count, len(mesh.edges), len(mesh.tets), len(mesh.surface_faces), len(mesh.pinned)) == \
            (392, 1831, 1170, 540, 98)

    def test_small_slab_bit_exact(self):
        mesh, rest, _ = build_slab_scene(with_attachments=True)
        g = golden("topology.npz")
        assert np.array_equal(mesh.tets, g["small_tets"])
        assert np.array_equal(mesh.edges, g["small_edges"])
        assert np.array_equal(mesh.surface_faces, g["small_faces"])
        assert np.array_equal(rest.rest_length, g["small_rest_length"])
        assert np.array_equal(rest.rest_volume, g["small_rest_volume"])

    def test_tet_soup_bit_exact(self):
        g = golden("topology.npz")
        e, f = derive_topology(g["soup_tets"])
        assert np.array_equal(e, g["soup_edges"]) and np.array_equal(f, g["soup_faces"])

    def test_shipped_scene_is_the_generated_preset(self, tmp_path, reach_scene_path):
        p = make_slab_scene(str(tmp_path), tets=1170, name="reach_1170")
        d = os.path.dirname(reach_scene_path)
        for f in ("reach_1170.scene", "reach_1170.mesh"):
            assert filecmp.cmp(os.path.join(tmp_path, f), os.path.join(d, f), shallow=False)
        assert os.path.basename(p) == "reach_1170.scene"


class TestTopology:
    def test_single_tet(self):
        edges, faces = derive_topology(np.array([[0, 1, 2, 3]]))
        assert len(edges) == 6 and len(faces) == 4

    def test_two_tets_sharing_face(self):
        edges, faces = derive_topology(np.array([[0, 1, 2, 3], [1, 2, 3, 4]]))
        assert len(edges) == 9 and len(faces) == 6
        assert (1, 2, 3) not in {tuple(sorted(f)) for f in faces.tolist()}

    def test_empty(self):
        edges, faces = derive_topology(np.zeros((0, 4), dtype=int))
        assert len(edges) == 0 and len(faces) == 0

    def test_edge_uniqueness_and_faces(self):
        rng = np.random.default_rng(0)
        for _ in range(20):
            tets = rng.integers(0, 30, size=(rng.integers(1, 40), 4))
            tets = tets[np.array([len(set(t)) == 4 for t in tets.tolist()])]
            if len(tets) == 0:
                continue
            edges, faces = derive_topology(tets)
            pairs = {tuple(e) for e in edges.tolist()}
            assert len(pairs) == len(edges) and all(a < b for a, b in pairs)
            assert {tuple(sorted(f)) for f in faces.tolist()} == surface_faces_oracle(tets)
            keys = [tuple(sorted(f)) for f in faces.tolist()]
            assert keys == sorted(keys)

    def test_slab_face_count(self):
        nx, ny, nz = 4, 2, 3
        pos, tets = make_slab(nx, ny, nz, 0.01)
        _, faces = derive_topology(fix_orientation(pos, tets))
        assert len(faces) == 4 * (nx * ny + ny * nz + nz * nx)

    def test_outward_winding(self):
        pos, tets = make_slab(2, 2, 2, 1.0)
        _, faces = derive_topology(fix_orientation(pos, tets))
        tri = pos[faces]
        normals = np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0])
        assert np.all(np.einsum("fk,fk->f", normals, tri.mean(axis=1) - pos.mean(axis=0)) > 0)

    def test_volumes(self):
        right = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
        assert signed_volumes(right, np.array([[0, 1, 2, 3]]))[0] == pytest.approx(1 / 6)
        assert signed_volumes(right, np.array([[0, 1, 3, 2]]))[0] == pytest.approx(-1 / 6)
        fixed = fix_orientation(right, np.array([[0, 1, 3, 2]]))
        assert signed_volumes(right, fixed)[0] > 0


class TestValidation:
    def test_bad_indices(self):
        pos = np.zeros((4, 3))
        with pytest.raises(ValidationError):
            build_mesh(pos, [[0, 1, 2, 4]])
        with pytest.raises(ValidationError):
            build_mesh(pos, [[0, 1, 1, 2]])
        with pytest.raises(ValidationError):
            build_mesh(np.eye(4, 3), [[0, 1, 2, 3]], pinned=[7])

    def test_degenerate_tet(self):
        pos = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [3, 0, 0]], float)
        mesh = build_mesh(pos, [[0, 1, 2, 3]])
        with pytest.raises(ValidationError):
            compute_rest_state(mesh)

    def test_config_ranges(self):
        for field, bad in (("dt", 0.0), ("substeps", 0), ("k_s", 1.5), ("damping", -1.0), ("clamp_angle", 30.0),
                           ("grasp_radius", 0.0), ("max_episode_steps", 0), ("action_scale", 0.0)):
            cfg = SceneConfig()
            setattr(cfg, field, bad)
            with pytest.raises(ValidationError):
                cfg.validate()


class TestParsing:
    def test_header_required(self):
        with pytest.raises(ParseError):
            parse_mesh_text("tetmesh 2\n1 0\n0 0 0\n")

    def test_counts_and_pins(self):
        pos, tets, pinned = parse_mesh_text("tetmesh 1\n4 1  # comment\n0 0 0\n1 0 0\n0 1 0\n0 0 1\n0 1 2 3\npinned 2 0 1\n")
        assert pos.shape == (4, 3) and tets.tolist() == [[0, 1, 2, 3]] and pinned == [0, 1]

    def test_bad_pinned_count(self):
        with pytest.raises(ParseError):
            parse_mesh_text("tetmesh 1\n4 1\n0 0 0\n1 0 0\n0 1 0\n0 0 1\n0 1 2 3\npinned 3 0 1\n")

    def test_unknown_scene_key(self):
        with pytest.raises(ParseError):
            parse_scene_text("bogus = 1\n")

    def test_vec3_needs_three(self):
        with pytest.raises(ParseError):
            parse_scene_text("rcm = 1 2\n")

    def test_missing_files(self, tmp_path):
        with pytest.raises(ParseError):
            load_scene(str(tmp_path / "nope.scene"))

    def test_round_trip(self, tmp_path, reach_scene):
        mesh, rest, cfg = reach_scene
        write_mesh(str(tmp_path / "m.mesh"), mesh.positions_rest, mesh.tets, mesh.pinned)
        cfg2 = SceneConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
        cfg2.mesh_path = str(tmp_path / "m.mesh")
        write_scene(str(tmp_path / "s.scene"), cfg2, mesh_name="m.mesh")
        m2, r2, c2 = load_scene(str(tmp_path / "s.scene"))
        assert np.array_equal(m2.edges, mesh.edges) and np.array_equal(r2.rest_volume, rest.rest_volume)
        assert c2.substeps == cfg.substeps and np.array_equal(c2.rcm, cfg.rcm)
