"""The operator CLI (host only) and POLAR_POLICY loading."""
import json
import os
import subprocess
import sys

from paper_2603_11438_b200 import cli
from paper_2603_11438_b200 import polar as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_validate_and_reject(capsys, tmp_path):
    assert cli.main(["validate", os.path.join(ROOT, "policies", "b200_virtual.json")]) == 0
    assert cli.main(["validate", os.path.join(ROOT, "policies", "nvlink_ring_mid_v2.json")]) == 0
    nvls = tmp_path / "nvls.json"
    nvls.write_text(json.dumps({"name": "nvls", "rows": [[0, 0, 1 << 30, 2, 2, 0]]}))
    assert cli.main(["validate", str(nvls)]) == 3
    assert "eunsupported" in capsys.readouterr().out
    L.set_policy([])


def test_explain_and_decide(capsys):
    assert cli.main(["explain", os.path.join(ROOT, "policies", "listing1_size_aware.json"), "--nranks", "8"]) == 0
    out = capsys.readouterr().out
    assert "32 KiB  tree" in out and "64 KiB  ring" in out
    assert cli.main(["decide", os.path.join(ROOT, "policies", "c1_fixed_threshold.json"), "--nranks", "2",
                     "--bytes", "65536"]) == 0
    d = json.loads(capsys.readouterr().out)
    assert (d["algo"], d["proto"], d["nchannels"]) == ("oneshot", "ll", 2)
    L.set_policy([])


def test_reload_and_adaptive(capsys):
    assert cli.main(["reload-test", "--calls", "40000", "--swaps", "100"]) == 0
    assert "PASS" in capsys.readouterr().out
    assert cli.main(["adaptive-sim"]) == 0
    tr = json.loads(capsys.readouterr().out)["channels_after_each_window"]
    assert tr[9] == 12 and max(tr[11:20]) <= 3 and tr[-1] == 12
    assert cli.main(["adaptive-sim", "--no-profiler"]) == 0
    assert set(json.loads(capsys.readouterr().out)["channels_after_each_window"]) == {2}
    L.set_policy([])


def test_polar_policy_env_loads_table(tmp_path):
    env = dict(os.environ)
    env["POLAR_POLICY"] = os.path.join(ROOT, "policies", "bad_channels.json")
    code = ("from paper_2603_11438_b200 import polar as L; d = L.decide(8, 1 << 27); "
            "print(d.nchannels, L.generation())")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.split() == ["1", "1"]
    nvls = tmp_path / "nvls.json"
    nvls.write_text(json.dumps({"name": "nvls", "rows": [[0, 0, 1 << 30, 2, 2, 0]]}))
    env["POLAR_POLICY"] = str(nvls)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "EUNSUPPORTED" in r.stderr
