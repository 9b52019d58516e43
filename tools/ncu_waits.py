"""Attribute warp-stall samples of an ncu --set full capture to mbarrier waits.

    python tools/ncu_waits.py <report.ncu-rep>

Each `@!P BRA <retry block>` whose target begins with a TRYWAIT (after an
optional YIELD) is charged to
that TRYWAIT's barrier operand, together with the samples of the retry block
itself; prints the barrier operands by samples, and the share of all samples.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = [r for r in csv.reader(io.StringIO(out))]
    rows = [r for r in rows if len(r) > 2 and r[0].startswith("0x")]
    idx = {r[0]: i for i, r in enumerate(rows)}
    samples = [int(r[2]) if r[2].isdigit() else 0 for r in rows]
    total = sum(samples)
    acc = {}

    def bar_of(i):
        src = rows[i][1]
        return src.split("[", 1)[1].split("]", 1)[0] if "TRYWAIT" in src else None

    for i, r in enumerate(rows):
        src = r[1]
        key = bar_of(i)
        if key:
            acc[key] = acc.get(key, 0) + samples[i]
        if "BRA 0x" in src:
            tgt = "0x" + src.split("BRA 0x", 1)[1].split()[0].rstrip(";")
            j = idx.get(tgt)
            if j is not None and "YIELD" in rows[j][1] and j + 1 < len(rows):
                j += 1  # retry blocks may start with a YIELD
            if j is not None and bar_of(j):
                acc[bar_of(j)] = acc.get(bar_of(j), 0) + samples[i]
    print(f"total samples {total}")
    for k, v in sorted(acc.items(), key=lambda x: -x[1])[:20]:
        print(f"{v:7d} {100.0 * v / max(total, 1):5.1f}%  {k}")


if __name__ == "__main__":
    main()
