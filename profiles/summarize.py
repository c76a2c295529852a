#!/usr/bin/env python
"""Summaries of ncu captures for profiles/ (run here, on CPU, after gpurun).

  python profiles/summarize.py launches <launches.csv> <out.md> [traffic.json key]
      per-kernel device time (serialised, cold-cache) and DRAM bytes of the library's
      kernels in the captured steps, their share of the step, bytes per launch.
  python profiles/summarize.py full <report.ncu-rep> <out.md>
      per-kernel key metrics of an `ncu --set full` capture (duration, DRAM bytes,
      throughput, occupancy, issue activity, top stall reasons).
"""
import collections
import csv
import json
import subprocess
import sys

OURS = ("k_count", "k_scan", "k_offsets", "k_scatter", "k_msd_tiles", "k_offsets_seg",
        "k_leaf", "k_copy", "k_keyhist", "k_validate", "k_tile_bounds", "k_block", "k_merge",
        "k_compress")


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("lco::", "")
    return n


def launches(path, out, traffic_key=None):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                             "Metric Unit"))
    idi = hdr.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        k = short(r[ki])
        if not any(k.startswith(o) for o in OURS):
            continue
        val = float(r[vi].replace(",", ""))
        unit = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            val = val / 1e3 if unit == "ns" else (val if unit == "us" else val * 1e3)
        per[r[idi]][r[mi]] = val
        names[r[idi]] = k
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    lines = ["| kernel | launches | total us | share | DRAM read B / launch | DRAM write B / launch |",
             "|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {a[0]} | {a[1]:.1f} | {100 * a[1] / tot:.1f}% | "
                     f"{a[2] / a[0]:.3e} | {a[3] / a[0]:.3e} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return {k: (a[2] + a[3]) / a[0] for k, a in agg.items()}


def marker_traffic(path, markers):
    """DRAM bytes (read + write) per launch of the kernel behind each bench marker.

    `markers` is one call's launch sequence (bench.py "markers"); the launch list's kernels
    of this library, in launch order, must repeat it exactly: each launch's kernel name
    (before the template arguments) must equal its marker or prefix it up to a "_"
    (k_scatter<10, ...> for k_scatter_seg).  Any mismatch raises instead of keying bytes
    to the wrong kernel.  Returns {marker: {"kernel": ncu name, "bytes": mean per launch}}."""
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value"))
    idi = hdr.index("ID")
    per = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        k = short(r[ki])
        if not k.startswith("k_"):
            continue
        per.setdefault(r[idi], {"name": k})[r[mi]] = float(r[vi].replace(",", ""))
    launches = list(per.values())
    if not markers or len(launches) % len(markers):
        raise ValueError(f"{len(launches)} launches do not repeat the {len(markers)} markers")
    out = collections.defaultdict(list)
    names = {}
    for j, l in enumerate(launches):
        m = markers[j % len(markers)]
        base = l["name"].split("<")[0]
        if not (m == base or m.startswith(base + "_")):
            raise ValueError(f"launch {j}: kernel {l['name']} does not match marker {m}")
        names[m] = l["name"]
        out[m].append(l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0))
    return {m: {"kernel": names[m], "bytes": sum(v) / len(v)} for m, v in out.items()}


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum", "launch__grid_size"]


def full(path, out):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        lines.append(f"### `{short(r[hdr.index('Kernel Name')])}`")
        for w in WANT:
            if w in hdr:
                lines.append(f"- {w}: {r[hdr.index(w)]} {units[hdr.index(w)]}")
        st = [(hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", ""), r[i])
              for i in range(len(hdr)) if "smsp__pcsamp_warps_issue_stalled" in hdr[i]
              and "not_issued" not in hdr[i]]
        st = sorted(((h, float(v)) for h, v in st if v.replace(".", "").isdigit()),
                    key=lambda x: -x[1])[:6]
        lines.append("- top stall samples: " + ", ".join(f"{h} {int(v)}" for h, v in st))
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        t = launches(sys.argv[2], sys.argv[3])
        if len(sys.argv) > 4:
            path = "profiles/traffic.json"
            try:
                d = json.load(open(path))
            except Exception:
                d = {}
            d[sys.argv[4]] = t
            json.dump(d, open(path, "w"), indent=1)
    else:
        full(sys.argv[2], sys.argv[3])
