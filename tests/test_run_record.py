"""Run records in the reference's report formats (SURVEY §8 f, row 3).

avec-loadgen writes client 0's timed cycles as a cycle CSV and a summary
markdown (paper_2103_04930_b200/csrc/host/record.cpp). The REFERENCE's own
parser (proj/src/profiler.cpp read_cycle_csv, via oracle/_ref/ref_record)
must accept the CSV, find the time decomposition consistent
(decomposition_holds) and render the very same summary markdown; per-cycle
byte counts must match the wire size law (transfer_size + 36 framing bytes,
proj/tests/test_client_server.cpp:488-503). CPU only: the product server
runs over the test-only CPU stub backend.
"""
import json
import pathlib
import subprocess

import pytest

import oracle_lib as O
import wire_client as W

ROOT = pathlib.Path(__file__).resolve().parent.parent
STUB = ROOT / "build" / "avec_stub_server"
LOADGEN = ROOT / "paper_2103_04930_b200" / "bin" / "avec-loadgen"
REF_RECORD = ROOT / "oracle" / "_ref" / "ref_record"


@pytest.fixture()
def server(tmp_path):
    if not STUB.exists():
        subprocess.run(["make", "-C", str(ROOT), "build/avec_stub_server"], check=True, stdout=subprocess.DEVNULL)
    srv = W.ServerProc([str(STUB), "--log", str(tmp_path / "events.jsonl")])
    yield srv
    srv.stop()


def _loadgen(endpoint, tmp_path, steps, w, h, batch):
    if not LOADGEN.exists():
        pytest.skip("avec-loadgen not built")
    csv, md = tmp_path / "run.csv", tmp_path / "run.md"
    r = subprocess.run([str(LOADGEN), "--endpoint", endpoint, "--clients", "1", "--steps", str(steps),
                        "--warmup", "1", "--batch", str(batch), "--width", str(w), "--height", str(h),
                        "--model", "mockpose", "--record-csv", str(csv), "--record-md", str(md),
                        "--label", "b200-test"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["ok"], out
    return csv, md


def test_csv_layout(server, tmp_path):
    csv, _ = _loadgen(server.endpoint, tmp_path, 5, 64, 32, 2)
    lines = csv.read_text().splitlines()
    meta = [l for l in lines if l.startswith("# ")]
    keys = [l[2:].split("=", 1)[0] for l in meta]
    assert keys == ["label", "mode", "host", "destination", "workload", "model", "output_divisor",
                    "scale_factor", "frames", "setup_s", "total_wall_s", "bytes_sent", "bytes_received",
                    "result_digest"]
    rows = lines[len(meta):]
    assert rows[0] == "index,gpu_s,communication_s,other_s,bytes_sent,bytes_received"
    assert len(rows) == 1 + 5
    dt = O.transfer_size(1, 3 * 2, 32, 64, 192.0 / 57.0)
    for i, row in enumerate(rows[1:]):
        c = row.split(",")
        assert int(c[0]) == i
        assert all(float(x) >= 0 for x in c[1:4])
        # FrameData + Resolution + FrameSize out, ForwardResult back: transfer_size + 36
        assert int(c[4]) + int(c[5]) == dt + 36


def test_reference_parser_accepts_and_renders_same_summary(server, tmp_path):
    if not REF_RECORD.exists():
        pytest.skip("reference tooling not built (needs /root/reference at build time)")
    csv, md = _loadgen(server.endpoint, tmp_path, 6, 80, 48, 1)
    r = subprocess.run([str(REF_RECORD), "--csv", str(csv)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    *ref_md, status = r.stdout.rstrip("\n").split("\n")
    st = json.loads(status)
    assert st["ok"] and st["frames"] == 6 and st["decomposition_holds"]
    # the reference renders our record exactly as we do
    assert "\n".join(ref_md) + "\n" == md.read_text()
