"""The elastik-compatible CLI (paper_2102_05221_b200.cli), mirroring the reference's
CLI tests (pkg/tests/test_cli.py): output formats, exit codes, and the answers of the
GPU path against the oracle.  Usage / configuration errors and `gen` run on CPU."""

import csv
import io
import json

import numpy as np
import pytest

from conftest import FIG_S, FIG_T
from oracle import eko
from paper_2102_05221_b200 import DistanceSpec, gen_random_walk, load_tsv, write_tsv
from paper_2102_05221_b200.cli import main

FIG_A = ",".join(str(v) for v in FIG_S)
FIG_B = ",".join(str(v) for v in FIG_T)


def run(capsys, *argv):
    code = main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


def jsonl(out):
    return [json.loads(line) for line in out.strip().splitlines()]


# ---------------------------------------------------------------- CPU: parsing and configuration

def test_usage_errors_exit_1(capsys):
    assert run(capsys)[0] == 1  # no subcommand
    code, _, err = run(capsys, "dist", "--kind", "warp", "--a", FIG_A, "--b", FIG_B)
    assert code == 1 and "error" in err
    code, _, err = run(capsys, "dist", "--kind", "dtw", "--b", FIG_B)  # --a missing
    assert code == 1 and "provide --a" in err
    code, _, err = run(capsys, "dist", "--kind", "cdtw", "--a", FIG_A, "--b", FIG_B)  # cdtw needs a window
    assert code == 1 and "window" in err
    code, _, err = run(capsys, "nn", "--kind", "msm", "--msm-c", "0.5", "--train", "x", "--test", "y", "--lb",
                       "keogh")
    assert code == 1
    code, _, err = run(capsys, "dist", "--kind", "dtw", "--a", FIG_A, "--b", FIG_B, "--precision", "half")
    assert code == 1


def test_missing_file_exit_1(capsys, tmp_path):
    code, _, err = run(capsys, "nn", "--kind", "dtw", "--train", str(tmp_path / "none.tsv"), "--test",
                       str(tmp_path / "none.tsv"))
    assert code == 1 and "error" in err


def test_gen_writes_reloadable_datasets(capsys, tmp_path):
    tr, te = tmp_path / "tr.tsv", tmp_path / "te.tsv"
    code, out, _ = run(capsys, "gen", "--gen-train", "6", "--gen-test", "4", "--gen-length", "20",
                       "--gen-classes", "3", "--seed", "11", "--out-train", str(tr), "--out-test", str(te))
    assert code == 0
    info = json.loads(out)
    assert info["train_count"] == 6 and info["test_count"] == 4 and info["length"] == 20
    a = load_tsv(str(tr))
    b = gen_random_walk(6, 20, 3, 11)
    assert [lab for lab, _ in a.entries] == [lab for lab, _ in b.entries]
    assert all(np.array_equal(x, y) for (_, x), (_, y) in zip(a.entries, b.entries))


# ---------------------------------------------------------------- GPU: answers

@pytest.mark.gpu
def test_dist_fig1_and_abandon(gpu, capsys):
    code, out, _ = run(capsys, "dist", "--kind", "dtw", "--a", FIG_A, "--b", FIG_B)
    assert code == 0
    p = json.loads(out)
    assert p["cost"] == 9.0 and p["cells_computed"] == 36 and p["config"]["backend"] == "cuda"
    code, out, _ = run(capsys, "dist", "--kind", "dtw", "--variant", "eapruned", "--cutoff", "6", "--a", FIG_A,
                       "--b", FIG_B)
    assert code == 2
    p = json.loads(out)
    assert p["cost"] == "abandoned" and abs(p["cells_computed"] - 20) <= 2
    code, out, _ = run(capsys, "dist", "--kind", "cdtw", "--window", "1", "--a", FIG_A, "--b", "1,2,3,4,5,6,7,8")
    assert code == 2 and json.loads(out)["cost"] == "abandoned"
    code, out, _ = run(capsys, "dist", "--kind", "dtw", "--a", FIG_A, "--b", FIG_B, "--precision", "float32")
    assert code == 0 and json.loads(out)["cost"] == 9.0


@pytest.mark.gpu
def test_nn_jsonl_matches_oracle(gpu, capsys, tmp_path):
    train = gen_random_walk(40, 64, 3, 5)
    test = gen_random_walk(12, 64, 3, 6)
    write_tsv(train, str(tmp_path / "tr.tsv"))
    write_tsv(test, str(tmp_path / "te.tsv"))
    code, out, _ = run(capsys, "nn", "--kind", "cdtw", "--window", "6", "--train", str(tmp_path / "tr.tsv"),
                       "--test", str(tmp_path / "te.tsv"))
    assert code == 0
    lines = jsonl(out)
    rows, summary = lines[:-1], lines[-1]
    assert summary["command"] == "nn" and summary["queries"] == 12
    spec = DistanceSpec(kind="cdtw", window=6)
    Q = [v for _, v in test.entries]
    C = [v for _, v in train.entries]
    r = eko.nn(spec, "eapruned", Q, C)
    labels = [lab for lab, _ in train.entries]
    assert [x["nn_index"] for x in rows] == r["nn_index"].tolist()
    assert [x["nn_distance"] for x in rows] == r["nn_distance"].tolist()
    assert [x["predicted"] for x in rows] == [labels[i] for i in r["nn_index"]]
    acc = np.mean([x["predicted"] == x["actual"] for x in rows])
    assert summary["accuracy"] == pytest.approx(acc)


@pytest.mark.gpu
def test_subseq_and_bench(gpu, capsys, tmp_path, rng):
    ref = np.cumsum(rng.normal(0, 1, 400))
    q = ref[123:163] + rng.normal(0, 0.01, 40)
    from paper_2102_05221_b200 import LabeledDataset

    write_tsv(LabeledDataset("q", ((0, q),)), str(tmp_path / "q.tsv"))
    write_tsv(LabeledDataset("r", ((0, ref),)), str(tmp_path / "r.tsv"))
    code, out, _ = run(capsys, "subseq", "--kind", "cdtw", "--window", "4", "--query", str(tmp_path / "q.tsv"),
                       "--reference", str(tmp_path / "r.tsv"), "--normalize")
    assert code == 0
    p = json.loads(out)
    want = eko.subsequence(DistanceSpec(kind="cdtw", window=4), "eapruned", q, ref, True)
    assert p["offset"] == want[0] == 123 and p["distance"] == want[1] and p["windows"] == 361
    code, out, _ = run(capsys, "bench", "--kind", "dtw", "--gen-train", "8", "--gen-test", "4", "--gen-length",
                       "32", "--reps", "2")
    assert code == 0
    table = list(csv.DictReader(io.StringIO(out)))
    assert [r["variant"] for r in table] == ["base", "ea", "eapruned", "pruned_only"] * 2
    assert len({r["accuracy"] for r in table}) == 1  # results are variant-invariant
    assert all(r["speedup_vs_base"] for r in table)
