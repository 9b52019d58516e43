"""Regenerate tests/golden/reference_golden.json from the REFERENCE library.

Runs oracle/_ref/ref_golden (our driver linking the reference's own sources,
built by `make -C oracle ref` from /root/reference/proj/src) and stores its JSON
output. Needs /root/reference, so it runs in the build container only; the
committed JSON is what the GPU box and the CPU suite check against.
"""
import json
import pathlib
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parent.parent


def main() -> int:
    subprocess.run(["make", "-C", str(ROOT / "oracle"), "ref"], check=True,
                   stdout=subprocess.DEVNULL)
    out = subprocess.run([str(ROOT / "oracle" / "_ref" / "ref_golden")], check=True,
                         capture_output=True, text=True).stdout
    data = json.loads(out)
    data["_generated_by"] = "oracle/_ref/ref_golden (reference accelfwd library)"
    (HERE / "reference_golden.json").write_text(json.dumps(data, indent=1) + "\n")
    print("wrote", HERE / "reference_golden.json")
    return 0


if __name__ == "__main__":
    sys.exit(main())
