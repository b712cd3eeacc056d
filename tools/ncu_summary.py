"""Summaries of the round's ncu outputs for profiles/.

    python tools/ncu_summary.py launches <launches.csv>      # per-kernel launch list
    python tools/ncu_summary.py full <full.ncu-rep> <json> [label] [source]
        # --set full digest; merges {label: per-stage DRAM bytes} into <json>

`launches`: the --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv list of one bench command, aggregated per kernel
(count, mean device time, mean DRAM bytes per launch).
`full`: per launch of a --set full capture: duration, DRAM bytes, throughput,
occupancy, issue activity and the top stall reasons; writes the per-stage DRAM
traffic (bytes per launch) that bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0,
         "msecond": 1e3, "second": 1e6}

STAGE_OF = {"k_corr_tiles": "corr_matvec", "k_k1_spmv": "near_project", "k_k1_lines": "near_project",
            "k_observers": "observers", "k_far_project": "far_project", "k_permute_q": "permute_q",
            "k_far_sum": "far_sum"}


def launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    iK, iM, iV, iU, iID = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        if len(r) <= iV:
            continue
        per[int(r[iID])][r[iM]] = float(r[iV].replace(",", "")) * SCALE.get(r[iU], 1.0)
        names[int(r[iID])] = r[iK].split("(")[0].replace("void ", "")
    agg = defaultdict(list)
    for i, m in per.items():
        agg[names[i]].append(m)
    out = ["# count  mean_us  mean_dram_MB  kernel   (ncu --clock-control none, serialised, cold cache)"]
    total = 0.0
    for k, ms in sorted(agg.items(), key=lambda x: -sum(m.get("gpu__time_duration.sum", 0) for m in x[1])):
        t = sum(m.get("gpu__time_duration.sum", 0) for m in ms) / len(ms)
        b = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in ms) / len(ms) / 1e6
        total += t * len(ms)
        out.append(f"{len(ms):6d} {t:9.2f} {b:12.2f}  {k}")
    out.append(f"# sum of device time over all launches: {total / 1e3:.2f} ms")
    print("\n".join(out))


RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "smsp__inst_executed.sum",
       "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "launch__grid_size", "launch__block_size"]


def full(rep, js, label="C2", source=None):
    if rep.endswith(".csv"):   # `ncu -i x.ncu-rep --page raw --csv` exported on the GPU box
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    iK = h.index("Kernel Name")
    traffic = {}
    print(f"# ncu --set full, {label} (bench.py --steps 2 --warmup 3 --no-cpu-baseline, FFTPIM_NO_GRAPHS=1)")
    print("# per launch: time us | DRAM MB (read+write) | DRAM % of peak | warps active % | regs | "
          "inst | L2 hit % | L1 % | issue % | grid x block | top stalls")
    for v in rows[2:]:
        def g(k):
            i = h.index(k)
            try:
                return float(v[i].replace(",", "")) * SCALE.get(units[i], 1.0)
            except ValueError:
                return float("nan")
        name = v[iK].split("(")[0].replace("void ", "")
        t = g("gpu__time_duration.sum")
        b = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
        stalls = sorted(((float(v[i].replace(",", "") or 0), k.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                         for i, k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled")
                         and not k.endswith("not_issued") and v[i].replace(",", "").replace(".", "").isdigit()),
                        reverse=True)[:3]
        print(f"{name:34s} {t:9.2f} | {b / 1e6:8.2f} | {g(RAW[3]):5.1f} | {g(RAW[4]):5.1f} | {g(RAW[5]):4.0f} | "
              f"{g(RAW[6]):.3g} | {g(RAW[7]):5.1f} | {g(RAW[8]):5.1f} | {g(RAW[9]):5.1f} | "
              f"{g(RAW[10]):.0f}x{g(RAW[11]):.0f} | " + ", ".join(f"{s[1]} {s[0]:.0f}" for s in stalls))
        for pre, stage in STAGE_OF.items():
            if name.startswith(pre) and stage not in traffic:
                traffic[stage] = int(b)
    try:
        doc = json.load(open(js))
    except (OSError, ValueError):
        doc = {}
    doc[label] = traffic
    doc.setdefault("sources", {})[label] = source or rep
    doc.setdefault("note", "dram__bytes_read.sum + dram__bytes_write.sum per launch, first launch of each stage kernel "
                           "in the --set full capture named in sources")
    doc.pop("source", None)
    json.dump(doc, open(js, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3], *sys.argv[4:6])
