"""Copy a milestone measurement (scripts/round_measure.sh outputs in gpurun_out/) into
profiles/ under a tag: bench JSON lines, ncu launch list + summaries, traffic per kernel."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1]
for c in ("C5", "C4", "C3a", "C3b", "C2a", "C2b", "C1"):
    src = os.path.join(G, f"m_bench_{c}.json")
    if os.path.exists(src) and os.path.getsize(src):
        shutil.copy(src, os.path.join(P, f"{tag}_bench_{c}.json"))
if os.path.exists(os.path.join(G, "m_ref_C5.json")):
    shutil.copy(os.path.join(G, "m_ref_C5.json"), os.path.join(P, f"{tag}_reference_C5.json"))
summ = os.path.join(P, "summarize.py")
if os.path.exists(os.path.join(G, "m_c5_launches.csv")):
    shutil.copy(os.path.join(G, "m_c5_launches.csv"), os.path.join(P, f"{tag}_c5_launches.csv"))
    subprocess.check_call([sys.executable, summ, "launches", os.path.join(G, "m_c5_launches.csv"),
                           os.path.join(P, f"{tag}_c5_launches.md")])
sys.path.insert(0, P)
import summarize  # noqa: E402

traffic = {}
# per bench marker (what bench.py's roofline.traffic looks up), from the launch lists
for c in ("C5", "C4", "C3a", "C3b", "C2a", "C2b", "C1"):
    lpath = os.path.join(G, f"m_{c.lower()}_launches.csv")
    bpath = os.path.join(G, f"m_bench_{c}.json")
    if os.path.exists(lpath) and os.path.exists(bpath):
        markers = json.load(open(bpath))["markers"]  # one call's launch sequence
        traffic[c] = summarize.marker_traffic(lpath, markers)
        if c != "C5":
            shutil.copy(lpath, os.path.join(P, f"{tag}_{c.lower()}_launches.csv"))
            subprocess.check_call([sys.executable, summ, "launches", lpath,
                                   os.path.join(P, f"{tag}_{c.lower()}_launches.md")])
for c, rep in (("C5", "m_c5_full.ncu-rep"), ("C4", "m_c4_full.ncu-rep")):
    path = os.path.join(G, rep)
    if not os.path.exists(path):
        continue
    out = os.path.join(P, f"{tag}_{c.lower()}_full.md")
    subprocess.check_call([sys.executable, summ, "full", path, out])
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    import csv
    rows = list(csv.reader(raw))
    h = rows[0]
    ki, r, w = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for row in rows[2:]:
        name = row[ki].split("(")[0].replace("void ", "").replace("lco::", "")
        b = float(row[r]) * scale.get(units[r], 1) + float(row[w]) * scale.get(units[w], 1)
        per.setdefault(name, []).append(b)
    # full-capture bytes by exact ncu kernel name (beside the per-marker launch-list bytes)
    traffic.setdefault(c, {})["by_kernel"] = {k: sum(v) / len(v) for k, v in per.items()}
tp = os.path.join(P, "traffic.json")
old = json.load(open(tp)) if os.path.exists(tp) else {}
for c, v in traffic.items():  # per config: keep entries this capture did not produce
    old.setdefault(c, {}).update(v)
json.dump(old, open(tp, "w"), indent=1)
for src, dst in (("m_table2.md", "table2.md"), ("m_table2.json", "table2.json"),
                 ("m_addition.json", "addition.json"), ("m_addition_hier.json", "addition_hier.json"),
                 ("m_mdt.json", "mdt.json")):
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, f"{tag}_{dst}"))
print("saved", tag, sorted(traffic))
