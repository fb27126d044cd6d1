"""Bench front end with the reference's report format (cli.py:22-128): CSV round trip, parser,
scene generation on CPU; a real (short) GPU bench row."""

import os

import numpy as np
import pytest

from paper_2503_18616_b200 import cli
from paper_2503_18616_b200.errors import ParseError


def test_report_csv_round_trip(tmp_path):
    rep = cli.BenchReport([cli.BenchRow(1, 1170, "sim", "b200", 14439.5, 12.25),
                           cli.BenchRow(65536, 52359, "sim", "b200", float("nan"), float("nan"), False)])
    p = tmp_path / "r.csv"
    rep.to_csv(p)
    assert p.read_text().splitlines()[0] == "envs,tets,mode,backend,mean_sps,std_sps,available"
    back = cli.BenchReport.from_csv(p)
    assert back.rows[0] == rep.rows[0]
    assert not back.rows[1].available and np.isnan(back.rows[1].mean_sps)
    assert "--" in back.pretty().splitlines()[2]


def test_report_rejects_other_files(tmp_path):
    p = tmp_path / "x.csv"
    p.write_text("a,b\n1,2\n")
    with pytest.raises(ParseError):
        cli.BenchReport.from_csv(p)


def test_make_scene_and_bad_counts(tmp_path, capsys):
    assert cli.main(["make-scene", "--tets", "1431", "--out", str(tmp_path)]) == 0
    path = capsys.readouterr().out.strip()
    assert os.path.exists(path) and path.endswith(".scene")
    assert cli.main(["bench", "--num-envs", "0"]) == 2


@pytest.mark.gpu
def test_bench_row_on_gpu(tmp_path):
    out = tmp_path / "bench.csv"
    assert cli.main(["bench", "--num-envs", "1,256", "--steps", "512", "--runs", "2", "--warmup", "3",
                     "--csv", str(out)]) == 0
    rep = cli.BenchReport.from_csv(out)
    assert [r.envs for r in rep.rows] == [1, 256]
    assert all(r.available and r.mean_sps > 0 and r.backend == "b200" for r in rep.rows)


def test_set_overrides_cast_like_the_reference():
    from paper_2503_18616_b200 import ppo
    from paper_2503_18616_b200.mesh import default_scene_path
    from paper_2503_18616_b200.errors import ValidationError
    pc = ppo.PPOConfig()
    mesh, rest, cfg = cli.load_scene_with_overrides(
        default_scene_path(), ["substeps=5", "k_v=0.5", "target=0.07 0.01 0.02", "ppo.learning_rate=1e-3",
                               "ppo.normalize_advantages=false", "ppo.hidden_sizes=64 64"], pc)
    assert cfg.substeps == 5 and cfg.k_v == 0.5 and np.array_equal(cfg.target, [0.07, 0.01, 0.02])
    assert pc.learning_rate == 1e-3 and pc.normalize_advantages is False and pc.hidden_sizes == (64, 64)
    for bad in (["substeps"], ["nosuch=1"], ["ppo.nosuch=1"]):
        with pytest.raises(ValidationError):
            cli.load_scene_with_overrides(default_scene_path(), bad, ppo.PPOConfig())
    with pytest.raises(ValidationError, match="k_v"):
        cli.load_scene_with_overrides(default_scene_path(), ["k_v=2"])


def test_parser_commands_and_errors(capsys):
    ap = cli.build_parser()
    a = ap.parse_args(["train", "--num-envs", "64", "--out", "x", "--set", "ppo.epochs=2", "--backend", "auto"])
    assert a.command == "train" and a.set_pairs == ["ppo.epochs=2"]
    a = ap.parse_args(["eval", "--checkpoint", "p.pt", "--episodes", "5"])
    assert a.command == "eval" and a.episodes == 5
    assert cli.main(["bench", "--backend", "numpy"]) == 2
    assert cli.main(["bench", "--set", "bogus=1"]) == 2
    assert "unknown scene setting" in capsys.readouterr().err


@pytest.mark.gpu
def test_train_then_eval_on_gpu(tmp_path, capsys):
    out = tmp_path / "run"
    assert cli.main(["train", "--num-envs", "64", "--steps", "2048", "--out", str(out), "--quiet",
                     "--set", "ppo.epochs=2"]) == 0
    assert (out / "policy.pt").exists() and (out / "train_log.csv").exists()
    assert "finished:" in capsys.readouterr().out
    assert cli.main(["eval", "--checkpoint", str(out / "policy.pt"), "--episodes", "8",
                     "--num-envs", "8"]) == 0
    assert "success rate" in capsys.readouterr().out
    assert cli.main(["eval", "--checkpoint", str(tmp_path / "missing.pt")]) == 2
