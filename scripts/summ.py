import json, sys, glob
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "ERR", e); continue
    c = d["config"]["workload"].split(":")[0]
    e2e = d.get("e2e") or {}
    print(f"{c:4s} {d['ms_per_step']:8.4f} ms {d['value']/1e9:7.2f} Gnnz/s step_frac {d['hbm_frac']:.3f} "
          f"dom {d['roofline']['kernel']} {d['roofline']['frac']:.3f} path {d['config']['plan']['path']} "
          f"e2e {e2e.get('value') and round(e2e['value']/1e9,3)} cpu {d.get('cpu_baseline') and round(d['cpu_baseline']['value']/1e6,2)}M")
    print("     ", {k: round(v, 3) for k, v in d["kernels_ms"].items()})
