"""Config-5 harness (tools/c5_replay, tools/lb_sim.*) on CPU.

1. Restatement parity: generate_trace / DualCache / tuner of the harness equal the reference's own
   code compiled from /root/reference (oracle/ref.mk -> oracle/_ref/libref_sim.a) on every record,
   lookup outcome, promotion, tail hit, window counter, gradient, alpha step and final resident
   order (tools/ref_parity.cpp).  Skipped where /root/reference is absent (the GPU box).
2. Latency composition pinned like the reference's own unit tests (proj/tests/test_sim.cpp:34-65):
   with a constant 40 ms decode, no batching and idle GPUs, a latent hit is served in 40 + 10 ms and
   a cold full miss in 140 + 40 + 10 ms; image hits cost the 10 ms network leg.
3. The full C5 workload replays in virtual time and reports a sane outcome mix and p50 <= p99.
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOLS = os.path.join(ROOT, "tools")


@pytest.fixture(scope="module")
def c5():
    from paper_2605_19385_b200 import build
    build.build()
    return build.build_tools()


def _run(exe, *args):
    out = subprocess.run([exe, *args], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj"), reason="reference sources not present")
@pytest.mark.parametrize("seed,sizes", [("7", "fixed"), ("11", "lognormal")])
def test_restatement_matches_reference(tmp_path, seed, sizes):
    subprocess.check_call(["make", "-s", "-f", "ref.mk"], cwd=os.path.join(ROOT, "oracle"))
    exe = str(tmp_path / "ref_parity")
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-I/root/reference/proj/include", "-I", TOOLS,
                           os.path.join(TOOLS, "ref_parity.cpp"), os.path.join(TOOLS, "lb_sim.cpp"),
                           os.path.join(ROOT, "oracle", "_ref", "libref_sim.a"), "-o", exe])
    out = subprocess.run([exe, seed, sizes[0]], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.startswith("OK"), out.stdout


def test_latency_composition_matches_reference_model(c5):
    d = _run(c5, "sim", "--days", "2", "--rpd", "20000", "--objects", "5000", "--gpus", "4096",
             "--max-batch", "1", "--max-wait-ms", "0", "--service", "40,80,160,320,640,1280", "--scale", "1")
    s = d["sim"]
    assert s["decode_p50_ms"] == 40.0 and s["decode_p99_ms"] == 40.0  # no queueing: pure service
    assert s["e2e_p50_ms"] == 10.0  # most requests are image hits: network leg only
    assert s["e2e_p99_ms"] == 190.0  # cold full miss: fetch 140 + decode 40 + net 10


def test_c5_full_workload_sim(c5):
    d = _run(c5, "sim", "--gpus", "8", "--scale", "10")
    assert d["requests"] == 10_000_000 and d["objects"] == 120_000
    mix = d["mix"]
    assert abs(mix["image_hit"] + mix["latent_hit"] + mix["full_miss"] + mix["coalesced"] - 1.0) < 1e-3
    assert 0.5 < mix["image_hit"] < 0.9 and 0.1 < mix["full_miss"] < 0.35
    s = d["sim"]
    assert 0 < s["decode_p50_ms"] <= s["decode_p99_ms"] and s["decodes"] > 1_000_000


def _ref_binding():
    p = os.path.join(ROOT, "oracle", "_ref", "ref_binding")
    if not os.path.exists(p):
        pytest.skip("oracle/_ref/ref_binding not built (needs /root/reference at build time)")
    return p


def test_reference_binding_runs_reference_simulator():
    """tools/ref_binding.cpp, compiled against the reference's own sources: the reference simulator
    (lbx::run) with LatencyModel::decode_ms swapped for a given decode time; fewer ms of decode
    means a lower tail; the outcome mix moves only through the split tuner (it observes T_decode)."""
    import json
    import subprocess
    out = subprocess.run([_ref_binding(), "--decode-ms", "9.0", "--requests-per-day", "50000", "--days", "4"],
                         capture_output=True, text=True, timeout=300, check=True).stdout
    lines = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    stock, ours = lines[1], lines[2]
    assert stock["decode_ms"] == 40.0 and ours["decode_ms"] == 9.0
    assert ours["e2e_p99_ms"] <= stock["e2e_p99_ms"] and ours["stage_decode_ms"] < stock["stage_decode_ms"]
    assert abs(ours["frac_full_miss"] - stock["frac_full_miss"]) < 0.01  # the tuner sees the new T_decode
