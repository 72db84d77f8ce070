"""Condense ncu output under gpurun_out/ into committed summaries under profiles/.

    python scripts/summarize_profiles.py r01

* launches_<cfg>.csv (the `--metrics gpu__time_duration.sum,dram__bytes_*` pass
  of bench.py) -> profiles/<round>_launches_<cfg>.csv: one row per launch with
  a short kernel name, duration and DRAM bytes; and the hot kernel's share.
* raw_/details_/source_<tag>.csv (a `--set full` capture) ->
  profiles/<round>_ncu_<tag>.txt: headline metrics + top stall reasons.
* profiles/ncu_traffic.json: DRAM bytes per launch of the hot kernel per
  config (bench.py reports it as roofline.traffic).
"""
import csv
import glob
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
HOT = {"C1": "tconv_outputs", "C2": "fold_ts_kernel", "C3": "wide_kernel", "C4": "ring_kernel", "C5": "wide_kernel"}


def short(name):
    m = re.search(r"segconv_b200::(?:\w+::)?(\w+)", name)
    base = m.group(1) if m else name.split("(")[0][-40:]
    t = re.search(r"<([^>]*)>", name)
    return base + (f"<{t.group(1)}>" if t and len(t.group(1)) < 40 else "")


def launches(rnd, cfg):
    path = os.path.join(G, rnd, f"launches_{cfg}.csv")
    if not os.path.exists(path):
        path = os.path.join(G, f"launches_{cfg}.csv")
    if not os.path.exists(path):
        return None
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    by = {}
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        by.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    out = []
    for (i, name), m in sorted(by.items(), key=lambda kv: int(kv[0][0])):
        out.append((int(i), short(name), m.get("gpu__time_duration.sum", 0.0),
                    m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)))
    with open(os.path.join(P, f"{rnd}_launches_{cfg}.csv"), "w") as f:
        f.write("id,kernel,duration_ns,dram_read_bytes,dram_write_bytes\n")
        for r in out:
            f.write(f"{r[0]},{r[1]},{r[2]:.0f},{r[3]:.0f},{r[4]:.0f}\n")
    ours = [r for r in out if not r[1].startswith("vectorized") and "elementwise" not in r[1]
            and "fill" not in r[1].lower()]
    hot = [r for r in ours if HOT[cfg] in r[1]]
    if hot and cfg == "C5":  # the stack's dominant kernel: layer a, the first pair-kernel launch of each step
        hot = [r for i, r in enumerate(hot) if i % 3 == 0]
    if hot:  # full-batch step launches only (the e2e leg launches per batch slice)
        big = max(r[2] for r in hot)
        hot = [r for r in hot if r[2] >= 0.5 * big]
    step = [r for r in ours if "segregate" not in r[1]]
    summary = {}
    if hot:
        avg = sum(r[2] for r in hot) / len(hot)
        summary = {"hot_kernel": hot[0][1], "launches": len(hot), "avg_duration_us": avg / 1e3,
                   "dram_bytes_per_launch": (hot[-1][3] + hot[-1][4]),
                   "avg_dram_bytes_per_launch": sum(r[3] + r[4] for r in hot) / len(hot),
                   "share_of_step_kernels": sum(r[2] for r in hot) / max(1e-9, sum(r[2] for r in step))}
    return summary


def full(rnd, tag):
    raw = os.path.join(G, f"raw_{tag}.csv")
    det = os.path.join(G, f"details_{tag}.csv")
    src = os.path.join(G, f"source_{tag}.csv")
    if not os.path.exists(raw):
        return None
    rows = list(csv.reader(open(raw)))
    d = dict(zip(rows[0], rows[2]))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "lts__t_bytes.sum", "smsp__inst_executed.sum"]
    lines = [f"# ncu --set full, {tag}  (kernel: {short(rows[2][rows[0].index('Kernel Name')]) if 'Kernel Name' in rows[0] else '?'})"]
    for k in keys:
        if k in d:
            lines.append(f"{k:70s} {d[k]}")
    if os.path.exists(det):
        drows = list(csv.reader(open(det)))
        h = drows[0]
        for r in drows[1:]:
            x = dict(zip(h, r))
            if x.get("Section Name") == "GPU Speed Of Light Throughput":
                lines.append(f"SOL {x['Metric Name']:40s} {x['Metric Value']} {x['Metric Unit']}")
    if os.path.exists(src):
        srows = list(csv.reader(open(src)))
        hdr = srows[1]
        stall = [i for i, hh in enumerate(hdr) if hh.startswith("stall_") and "Not Issued" not in hh]
        agg = {}
        for r in srows[2:]:
            for i in stall:
                agg[hdr[i]] = agg.get(hdr[i], 0.0) + float(r[i] or 0)
        tot = sum(agg.values()) or 1
        lines.append("warp stall samples (share): " + ", ".join(
            f"{k[6:]} {v / tot:.0%}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:6]))
        sass = [r[1] for r in srows[2:]]
        lines.append("SASS evidence: " + ", ".join(
            f"{m} x{sum(1 for s in sass if m in s)}" for m in ("UTCHMMA", "UTCBAR", "LDTM", "UTMALDG",
                                                               "UBLKCP", "SYNCS")))
    with open(os.path.join(P, f"{rnd}_ncu_{tag}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    return d


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(P, exist_ok=True)
    traffic_path = os.path.join(P, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for cfg in ("C1", "C2", "C3", "C4", "C5"):
        sm = launches(rnd, cfg)
        if sm:
            print(cfg, sm)
            traffic[cfg] = {"dram_bytes_per_launch": sm["dram_bytes_per_launch"],
                            "hot_kernel": sm["hot_kernel"],
                            "avg_duration_us_cold_serialised": sm["avg_duration_us"],
                            "share_of_step_kernels": sm["share_of_step_kernels"],
                            "source": f"profiles/{rnd}_launches_{cfg}.csv (ncu, cold cache)"
                            + (" -- layer a, the first of the stack's three pair-kernel launches per step"
                               if cfg == "C5" else "")}
    for f in glob.glob(os.path.join(G, "raw_*.csv")):
        tag = os.path.basename(f)[4:-4]
        if tag.endswith(rnd):
            full(rnd, tag)
    json.dump(traffic, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    main()
