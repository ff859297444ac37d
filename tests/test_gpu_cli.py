"""The CLI (cli.py:41-84 mirror) end to end on the GPU: UCR input -> report, outputs, exit codes."""

from __future__ import annotations

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _write_ucr(path, x, labels):
    with open(path, "w") as fh:
        for lab, row in zip(labels, x):
            fh.write("\t".join([str(int(lab))] + [repr(float(v)) for v in row]) + "\n")


def test_cli_runs_pipeline_and_writes_outputs(tmp_path, capsys):
    from paper_2408_09399_b200 import cli, load_dendrogram, serialize_dendrogram, synth
    x, labels = synth.generate(1, n=300)
    _write_ucr(tmp_path / "d.tsv", x, labels)
    rc = cli.main(["--input", str(tmp_path / "d.tsv"), "--apsp", "hub", "--out", str(tmp_path / "out")])
    assert rc == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["n"] == 300 and rep["k"] == int(labels.max()) + 1 and rep["ari"] is not None
    assert set(rep["stage_seconds"]) == {"initial_faces", "sorting", "tmfg_insertion", "apsp", "dbht", "linkage"}
    d = load_dendrogram(tmp_path / "out" / "dendrogram.txt")
    import hashlib
    assert hashlib.sha256(serialize_dendrogram(d).encode()).hexdigest() == rep["digest"]
    assert len((tmp_path / "out" / "labels.txt").read_text().split()) == 300
    rc = cli.main(["--input", str(tmp_path / "d.tsv"), "--compare", "exact,corr,heap", "--k", "5",
                   "--out", str(tmp_path / "cmp")])
    assert rc == 0
    rows = json.loads((tmp_path / "cmp" / "comparison.json").read_text())
    assert [r["variant"] for r in rows] == ["exact", "corr", "heap"]
    assert rows[0]["edge_sum_delta"] == 0.0


def test_cli_exit_codes(tmp_path):
    from paper_2408_09399_b200 import cli
    assert cli.main(["--input", str(tmp_path / "missing.tsv")]) == 2           # OSError
    (tmp_path / "bad.tsv").write_text("1\t0.1\t0.2\n2\t0.3\n")
    assert cli.main(["--input", str(tmp_path / "bad.tsv")]) == 2               # DataError (ragged)
    S = np.full((6, 6), 0.2)
    np.fill_diagonal(S, 1.0)
    S[1, 2] = S[2, 1] = 1.5                                                      # out of range -> stage error
    from paper_2408_09399_b200 import write_matrix_binary
    write_matrix_binary(tmp_path / "m.bin", S)
    assert cli.main(["--input", str(tmp_path / "m.bin"), "--format", "matrix", "--k", "2"]) in (1, 2)
