"""Summarize ncu captures into profiles/ (markdown + JSON).

usage: python tools/ncu_summary.py full <report.ncu-rep | raw.csv> <out.md> [--traffic-config N]
       python tools/ncu_summary.py launches <launches.csv> <out.md>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

KEYS = [
    ("gpu__time_duration.sum", "duration (ms)", 1e-6 if False else 1.0),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active %", 1.0),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %", 1.0),
    ("dram__bytes_read.sum", "DRAM read", 1.0),
    ("dram__bytes_write.sum", "DRAM write", 1.0),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1.0),
    ("launch__registers_per_thread", "regs/thread", 1.0),
    ("launch__grid_size", "grid", 1.0),
    ("launch__block_size", "block", 1.0),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1.0),
]


def raw_rows(rep):
    if str(rep).endswith(".csv"):  # `ncu -i ... --page raw --csv` exported on the GPU box
        out = Path(rep).read_text()
        out = out[out.find('"ID"'):]
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def full(rep, out_md, traffic_cfg=None):
    hdr, units, rows = raw_rows(rep)
    H = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary: `{Path(rep).name}`", "",
             "| # | kernel | " + " | ".join(k[1] for k in KEYS) + " |",
             "|---|---|" + "---|" * len(KEYS)]
    recs = []
    for i, r in enumerate(rows):
        name = r[H["Kernel Name"]]
        short = name.split("<", 2)[-1][:70] if "<" in name else name[:70]
        vals = []
        rec = {"kernel": name}
        for key, label, _ in KEYS:
            v = r[H[key]] if key in H else ""
            u = units[H[key]] if key in H else ""
            if key.startswith("dram__bytes") and v:
                f = float(v.replace(",", ""))
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                rec[key] = f * scale
                vals.append(f"{f * scale / 1e9:.3f} GB")
            else:
                rec[key] = v
                vals.append(f"{v} {u}".strip())
        recs.append(rec)
        lines.append(f"| {i} | `{short}` | " + " | ".join(vals) + " |")
    Path(out_md).write_text("\n".join(lines) + "\n")
    if traffic_cfg is not None:
        tf = Path("profiles/ncu_traffic.json")
        data = json.loads(tf.read_text()) if tf.exists() else {}
        top = max(recs, key=lambda q: float(str(q["gpu__time_duration.sum"]).replace(",", "") or 0))
        data[str(traffic_cfg)] = round(top["dram__bytes_read.sum"] + top["dram__bytes_write.sum"])
        tf.write_text(json.dumps(data, indent=1) + "\n")
    print("\n".join(lines))


def launches(csv_path, out_md):
    text = Path(csv_path).read_text()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r["Metric Unit"], 1e-6)
        name = r["Kernel Name"]
        short = name.split("(")[0][-90:]
        agg[short][0] += 1
        agg[short][1] += v * scale
        total += v * scale
    lines = [f"# ncu launch list (gpu__time_duration.sum, --clock-control none): `{Path(csv_path).name}`", "",
             "Cold-cache, serialized replays: compare shares, not absolute times.", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {ms:.3f} | {ms / total:.1%} |")
    Path(out_md).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        cfg = int(sys.argv[sys.argv.index("--traffic-config") + 1]) if "--traffic-config" in sys.argv else None
        full(sys.argv[2], sys.argv[3], cfg)
    else:
        launches(sys.argv[2], sys.argv[3])
