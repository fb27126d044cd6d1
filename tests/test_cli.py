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
