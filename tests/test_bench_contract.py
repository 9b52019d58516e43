"""bench.py's output contract (the driver parses it): one JSON line on stdout
with the required keys, for our arm and for the reference arm."""
import json
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks", "roofline", "cpu_baseline"]


def run_bench(*args):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout[-2000:]  # exactly one line, and it is JSON
    return json.loads(lines[0])


@pytest.mark.gpu
def test_our_arm_line():
    d = run_bench("--steps", "3", "--warmup", "3")
    for k in REQUIRED:
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert d["config"]["workload"].startswith("C2")
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * 3 * 656 * 368 * 4
    assert e["d2h_bytes_per_step"] == 8 * 57 * 46 * 82 * 4
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r
    assert 0 < r["frac"] < 1.5
    c = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c
    assert d["gpu_launches"] >= 3 * 40  # every step is one graph of the net's launches
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    # the other BASELINE configs ride in the same line
    assert d["steady_state"]["steps"] >= 200 and d["steady_state"]["value"] > 0
    assert d["roofline"]["peak_kind"].startswith("measured burst") or "burst" in d["roofline"]["peak_kind"]
    assert d["c1"]["ok"] and d["c1"]["byte_account_bad"] == 0 and d["c1"]["lat_ms_p90"] > 0
    assert d["mockpose_wire"]["ok"] and d["mockpose_wire"]["fps"] > 0
    assert all(x["exact"] for x in d["c3_memcpy"]["abi_pinned"]) and len(d["c3_memcpy"]["wire"]) == 8
    assert d["c4"]["ok"] and d["c4"]["clients"] == 8
    assert d["c5"]["value"] > 0 and d["c5"]["frames_per_step"] == 32


def test_reference_arm_line():
    # CPU only: the reference's own Server + MockPose + Session (oracle/_ref/ref_arm)
    if not (ROOT / "oracle" / "_ref" / "ref_arm").exists():
        pytest.skip("reference drivers not built")
    d = run_bench("--impl", "reference", "--steps", "3", "--warmup", "3")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
