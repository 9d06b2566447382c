"""bench.py's reference arm picks the same workload as our arm (config 2 at N = 1, config 4 at N > 1)
and prints the contract's keys; the CPU decode itself is stubbed (it takes tens of seconds)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.parametrize("gpus,fam,cfg", [(1, "sd15", "config2"), (8, "sd3", "config4")])
def test_reference_arm_workload(monkeypatch, capsys, gpus, fam, cfg):
    import bench
    seen = []

    def fake_sample(f, c, threads, seed=0):
        seen.append((f, c))
        return 0.5

    monkeypatch.setattr(bench, "cpu_decode_sample", fake_sample)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", str(gpus), "--steps", "2",
                                      "--warmup", "1"])
    monkeypatch.delenv("RANK", raising=False)
    args = bench.parse()
    assert bench.run_reference(args) == 0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == gpus
    assert line["config"]["workload"].startswith(cfg) and line["config"]["family"] == fam
    assert all(f == fam for f, _ in seen)
    assert line["value"] == pytest.approx(2.0) and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
