"""Sweep driver, report formats, CSV ingestion and dataset generators
(paper_1206_6857_b200.cli_harness / datasets vs the reference's cli_harness.py
and datasets.py).  Formats, loader outcomes and generator outputs are pinned
by tests/golden/cli.json, rendered by the unmodified reference
(tests/golden/make_golden.py cli)."""

import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(HERE, "golden", "cli.json")) as fh:
        return json.load(fh)


def _report(ch, entry):
    rows = [ch.SweepRow(a, m, h, s, e, c) for a, m, h, s, e, c in entry["rows"]]
    return ch.SweepReport(0.1, 0.01, "ref.csv", None, (0.5, 1.0), ("naive", "dfd"), rows,
                          entry["totals"], entry["verified"])


def test_report_formats_match_reference(gold):
    from paper_1206_6857_b200 import cli_harness as ch

    for entry in gold["reports"]:
        rep = _report(ch, entry)
        assert ch._format_table(rep) == entry["table"]
        assert ch._format_csv(rep) == entry["csv"]
        assert json.dumps(ch.report_to_dict(rep), indent=2) + "\n" == entry["json"]


def test_emit_report(gold, tmp_path, capsys):
    from paper_1206_6857_b200 import cli_harness as ch

    rep = _report(ch, gold["reports"][0])
    out = tmp_path / "r.csv"
    assert ch.emit_report(rep, "csv", str(out)) == out.read_text()
    ch.emit_report(rep, "table")
    assert capsys.readouterr().out == gold["reports"][0]["table"]
    with pytest.raises(ValueError):
        ch.emit_report(rep, "xml")
    with pytest.raises(ch.LoadError):
        ch.emit_report(rep, "json", str(tmp_path / "missing" / "r.json"))


def test_load_points_matches_reference(gold, tmp_path):
    from paper_1206_6857_b200 import cli_harness as ch

    path = tmp_path / "data.csv"
    for case in gold["loads"]:
        path.write_text(case["text"])
        if "error" in case:
            with pytest.raises(ch.LoadError) as exc:
                ch.load_points(str(path), **case["kw"])
            assert str(exc.value).replace(str(path), "<path>") == case["error"], case["name"]
        else:
            st = ch.load_points(str(path), **case["kw"])
            np.testing.assert_array_equal(st.points, np.array(case["points"]))
            np.testing.assert_array_equal(st.weights, np.array(case["weights"]))
    with pytest.raises(ch.LoadError):
        ch.load_points(str(tmp_path / "nope.csv"))


def test_dataset_generators_match_reference(gold):
    from paper_1206_6857_b200 import datasets as ds

    g = gold["datasets"]
    np.testing.assert_array_equal(ds.uniform_points(5, 3, 7), np.array(g["uniform"]))
    np.testing.assert_array_equal(ds.clustered_points(6, 2, 3), np.array(g["clustered"]))
    np.testing.assert_array_equal(ds.hierarchical_clusters(6, 2, 4), np.array(g["hierarchical"]))
    np.testing.assert_array_equal(ds.duplicated_points(10, 2, 5), np.array(g["duplicated"]))


def test_cli_usage_and_gen(tmp_path):
    from paper_1206_6857_b200 import cli_harness as ch
    from paper_1206_6857_b200.datasets import uniform_points

    assert ch.main([]) == 1
    with pytest.raises(SystemExit) as exc:
        ch.main(["sweep"])  # --ref missing
    assert exc.value.code == 1
    assert ch.main(["sweep", "--ref", str(tmp_path / "missing.csv"), "--h-star", "0.1"]) == 1
    assert ch.main(["sweep", "--ref", str(tmp_path / "missing.csv"), "--algos", "bogus"]) == 1
    out = tmp_path / "u.csv"
    assert ch.main(["gen", "--dist", "uniform", "--n", "50", "--dim", "3", "--out", str(out),
                    "--seed", "4"]) == 0
    st = ch.load_points(str(out))
    np.testing.assert_array_equal(st.points, uniform_points(50, 3, 4))
    with pytest.raises(ValueError):
        ch.SweepSpec(ref_path="x", multipliers=())
    with pytest.raises(ValueError):
        ch.SweepSpec(ref_path="x", algorithms=("fast",))


@pytest.mark.gpu
def test_sweep_end_to_end(tmp_path):
    from paper_1206_6857_b200 import cli_harness as ch
    from paper_1206_6857_b200.datasets import clustered_points

    ref = tmp_path / "ref.csv"
    np.savetxt(ref, clustered_points(3000, 3, 1), delimiter=",", fmt="%.17g")
    out = tmp_path / "rep.json"
    code = ch.main(["sweep", "--ref", str(ref), "--h-star", "0.05", "--multipliers", "0.1,1,10",
                    "--algos", "naive,dfd,dfdo,dito", "--verify", "--format", "json",
                    "--out", str(out)])
    assert code == 0
    rep = json.loads(out.read_text())
    assert [(r["algorithm"], r["multiplier"]) for r in rep["rows"]] == [
        (a, m) for m in (0.1, 1.0, 10.0) for a in ("naive", "dfd", "dfdo", "dito")]
    for r in rep["rows"]:
        assert r["max_rel_error"] <= 0.01
        assert r["seconds"] > 0.0
        assert r["bandwidth"] == pytest.approx(0.05 * r["multiplier"], rel=1e-15)
    for alg in ("naive", "dfd", "dfdo", "dito"):
        assert rep["totals"][alg] == pytest.approx(
            sum(r["seconds"] for r in rep["rows"] if r["algorithm"] == alg))
    # automatic h* (LSCV on the device) and the table format
    spec = ch.SweepSpec(ref_path=str(ref), multipliers=(1.0,), algorithms=("dito",), verify=True)
    report = ch.run_sweep(spec)
    assert report.h_star > 0.0 and report.worst_error <= 0.01
