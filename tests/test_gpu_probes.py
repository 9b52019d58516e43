"""tcgen05 / TMA probes (tests/native/tc_probe.cu, tc2_probe.cu, tma3d_probe.cu): the descriptor /
instruction-descriptor encodings the conv kernels rely on produce exact
GEMMs (single CTA and CTA pair), and the measured MMA rates the kernel
choices in DESIGN.md §3 are built on still hold."""
import json
import pathlib
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parent.parent


def run_probe(name):
    exe = ROOT / "build" / name
    if not exe.exists():
        subprocess.run(["make", "-C", str(ROOT), f"build/{name}"], check=True, stdout=subprocess.DEVNULL)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_single_cta_probe():
    d = run_probe("tc_probe")
    assert d["ok"]
    # with the descriptor's base-offset field left 0, any row offset is exact
    # (the kernels' sliding windows rely on it); the probe also records the
    # variants that set the field, which the kernels do not use
    assert all(c["bad"] == 0 for c in d["correctness"] if c["base_off_field"] == 0)
    rate = {x["N"]: x["cycles_per_mma"] for x in d["rate"]}
    assert rate[256] < 128 * 1.05 and rate[128] < 64 * 1.05  # full rate from N = 128
    assert rate[64] > 40  # N = 64 is operand-read bound (48 cycles, not 32)


def test_cta_pair_probe():
    d = run_probe("tc2_probe")
    assert d["ok"]
    assert all(c["bad"] == 0 for c in d["correctness"])
    rate = {x["N"]: x["cycles_per_mma"] for x in d["rate"]}
    assert rate[256] < 128 * 1.05 and rate[128] < 64 * 1.05
    assert rate[96] < 56  # the pair lifts N = 96 off the single-CTA 56-cycle operand bound


@pytest.mark.parametrize("c0,c1", [(0, 0), (-4, -2), (124, 5), (-4, 62)])
def test_tma_fp32_patch_probe(c0, c1):
    """The conv12 frame-patch load (tests/native/tma3d_probe.cu): a 3D fp32
    TMA box {132, 6, 3} with zero fill outside the frame is exact whenever the
    inner coordinate is a multiple of 4 floats (16 bytes), negative included.
    (An inner coordinate that is not — e.g. -2 — faults with an illegal
    instruction, which is why conv12 starts its patch at (x0 - 2) & ~3.)"""
    exe = ROOT / "build" / "tma3d_probe"
    if not exe.exists():
        subprocess.run(["make", "-C", str(ROOT), "build/tma3d_probe"], check=True, stdout=subprocess.DEVNULL)
    r = subprocess.run([str(exe), "200", "64", "6", "132", "6", "3", str(c0), str(c1), "3", "0"],
                       capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert json.loads(r.stdout.strip().splitlines()[-1])["ok"]
