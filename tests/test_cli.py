"""The command line vs the reference's own CLI output (tests/golden/cli.json,
produced by the reference's cli.main; its tests: test_cli.py:30-115).

CPU: `bitdiff` on the reference's run logs (IDENTICAL / first divergence /
shape mismatch = usage error), exit codes and the control-plane stubs.
GPU: `train` writes run logs and checkpoints byte-identical to the
reference's, and `reprocheck` prints the reference's report for d0/d1/d1d2.
"""

import pytest
import yaml

from golden_util import load

DOC = load("cli.json")


def _train_case(name):
    return next(c for c in DOC["train"] if c["name"] == name)


def _run(capsys, argv):
    from paper_2208_14228_b200.cli import main

    rc = main(argv)
    cap = capsys.readouterr()
    return rc, cap.out, cap.err


def test_bitdiff_on_reference_logs(tmp_path, capsys):
    paths = {}
    for c in DOC["train"]:
        paths[c["name"]] = tmp_path / f"{c['name']}.log"
        paths[c["name"]].write_text(c["log"], encoding="utf-8")
    for b in DOC["bitdiff"]:
        rc, out, err = _run(capsys, ["bitdiff", str(paths[b["a"]]), str(paths[b["b"]])])
        assert rc == b["rc"]
        assert out == b["stdout"]
        if rc == 2:
            assert err.startswith("error: ")


def test_missing_and_bad_inputs_are_usage_errors(tmp_path, capsys):
    rc, _, err = _run(capsys, ["bitdiff", str(tmp_path / "nope.log"), str(tmp_path / "nope2.log")])
    assert rc == 2 and err.startswith("error: ")
    bad = tmp_path / "bad.yaml"
    bad.write_text("seed: [\n", encoding="utf-8")
    rc, _, err = _run(capsys, ["train", "--config", str(bad), "--out", str(tmp_path / "x.log")])
    assert rc == 2 and "invalid YAML" in err
    with pytest.raises(SystemExit) as exc:
        _run(capsys, ["reprocheck", "--mode", "d9", "--matrix", "m.yaml"])
    assert exc.value.code == 2


def test_control_plane_commands_are_not_in_this_build(capsys):
    rc, _, err = _run(capsys, ["plan", "--pool", "p.yaml", "--profile", "q.yaml", "--maxp", "4"])
    assert rc == 2 and "control plane" in err
    rc, _, err = _run(capsys, ["simulate", "--trace", "t.csv", "--pool", "p.yaml", "--mode", "homo", "--out", "o"])
    assert rc == 2 and "control plane" in err


@pytest.mark.gpu
@pytest.mark.parametrize("name", [c["name"] for c in DOC["train"]])
def test_train_log_and_checkpoint_bytes_match_reference(tmp_path, capsys, name):
    c = _train_case(name)
    cfg = tmp_path / "cfg.yaml"
    cfg.write_text(yaml.safe_dump(c["doc"]), encoding="utf-8")
    log, ck = tmp_path / "run.log", tmp_path / "final.ckpt"
    rc, out, _ = _run(capsys, ["train", "--config", str(cfg), "--out", str(log), "--ckpt", str(ck)])
    assert rc == c["rc"] == 0
    assert out == c["stdout"]
    assert log.read_text(encoding="utf-8") == c["log"]
    assert ck.read_bytes().hex() == c["ckpt"]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["d0", "d1", "d1d2"])
def test_reprocheck_report_matches_reference(tmp_path, capsys, mode):
    r = next(x for x in DOC["reprocheck"] if x["mode"] == mode)
    m = tmp_path / "matrix.yaml"
    m.write_text(yaml.safe_dump(r["matrix"]), encoding="utf-8")
    rc, out, _ = _run(capsys, ["reprocheck", "--mode", mode, "--matrix", str(m)])
    assert rc == r["rc"]
    assert out == r["stdout"]
