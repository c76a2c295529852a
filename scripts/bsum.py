"""One-line summaries of bench JSON lines: python scripts/bsum.py gpurun_out/q_bench_*.json"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as ex:  # noqa: BLE001
        print(f, "unreadable", ex)
        continue
    r, sr = d["roofline"], d["step_roofline"]
    print(f"{f.split('/')[-1]}: {d['ms_per_step']:.4f} ms  step frac {sr['frac']:.3f}  dom "
          f"{r['kernel']} {r['launch_ms']:.3f} ms frac {r['frac']:.3f}  no_perm "
          f"{d.get('no_perm', {}).get('ms_per_step', 0):.4f}")
    print("   ", {k: v for k, v in d["kernels_ms"].items()})
