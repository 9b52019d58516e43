"""Summarise tools/ab.sh output: python tools/ab_report.py old new"""
import json, sys, pathlib
d = pathlib.Path(__file__).resolve().parent.parent / "gpurun_out"
for v in sys.argv[1:]:
    for r in (1, 2):
        for c in ("c2", "c5"):
            try:
                lt = json.loads((d / f"ab_lt_{v}_{r}_{c}.json").read_text())
                b = json.loads((d / f"ab_b_{v}_{r}_{c}.json").read_text())
                print(f"{v:6s} r{r} {c}: layer-table step {lt['step_ms']:.3f} ms | bench {b['value']:.1f} fps "
                      f"e2e {b['e2e']['value']:.1f} wire {b['wire'].get('fps', 0):.0f} sm {b['clocks']['sm_mhz']}")
            except Exception as e:  # noqa: BLE001
                print(v, r, c, "missing", e)
