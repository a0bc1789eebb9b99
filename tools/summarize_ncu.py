"""Summarise ncu reports (.ncu-rep) and launch lists into profiles/<round>/.

    python tools/summarize_ncu.py <round-tag> gpurun_out/prof_*.ncu-rep [--launches csv]

Writes profiles/<tag>/ncu_summary.md (one section per report: duration, DRAM
bytes, pipe utilisation, occupancy, divergence, top stall reasons) and
profiles/<tag>/launches.md (per-kernel launch counts / device time shares).
"""

import csv
import io
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

DETAILS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
           "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Registers Per Thread",
           "Theoretical Occupancy", "Achieved Occupancy", "Grid Size", "Block Size",
           "Avg. Active Threads Per Warp", "Warp Cycles Per Issued Instruction",
           "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate", "SM Frequency"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "smsp__thread_inst_executed_per_inst_executed.ratio",
       "launch__registers_per_thread"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize(rep):
    lines = [f"### {os.path.basename(rep)}", ""]
    rows = ncu_csv(rep, "details")
    if rows:
        hdr = rows[0]
        kname = None
        for r in rows[1:]:
            d = dict(zip(hdr, r))
            kname = kname or d.get("Kernel Name")
            if d.get("Metric Name") in DETAILS:
                lines.append(f"- {d['Metric Name']}: {d['Metric Value']} {d['Metric Unit']}")
        lines.insert(1, f"kernel: `{kname}`")
    raw = ncu_csv(rep, "raw")
    if len(raw) > 2:
        hdr, units, vals = raw[0], raw[1], raw[2]
        m = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        lines.append("")
        for k in RAW:
            if k in m:
                lines.append(f"- `{k}` = {m[k]} {u.get(k, '')}")
        stalls = sorted(((float(v.replace(',', '') or 0), h) for h, v in m.items()
                         if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                         and not h.endswith("_not_issued") and v.replace(',', '').replace('.', '').isdigit()),
                        reverse=True)[:6]
        if stalls:
            lines.append("- top stall samples: " + ", ".join(
                f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={int(v)}" for v, h in stalls))
    lines.append("")
    return "\n".join(lines)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            agg[d["Kernel Name"].split("(")[0]][0] += 1
            agg[d["Kernel Name"].split("(")[0]][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(t for _, t in agg.values()) or 1.0
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
    return "\n".join(lines) + "\n"


def main():
    tag = sys.argv[1]
    args = sys.argv[2:]
    lcsv = None
    if "--launches" in args:
        i = args.index("--launches")
        lcsv = args[i + 1]
        del args[i:i + 2]
    outdir = os.path.join(ROOT, "profiles", tag)
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, "ncu_summary.md"), "w") as fh:
        fh.write(f"# ncu --set full summaries ({tag})\n\n")
        fh.write("Captured with `ncu --set full --clock-control none --import-source on` on one "
                 "B200 via tools/gpu_profile.sh (driver: tools/prof_driver.py).\n\n")
        for rep in args:
            fh.write(summarize(rep) + "\n")
    # traffic per algorithmic byte for the HBM-bound kernels (bench.py reads it)
    alg = {"uniform": ("fill_uniform", 4096 * 65536 * 8 + (1 << 20) * 96),
           "normal": ("fill_normal_fast", (31250 // 8) * 32000 * 4 + (1 << 18) * 96)}
    traffic = {}
    for rep in args:
        for key, (kname, abytes) in alg.items():
            if f"prof_{key}_" in os.path.basename(rep):
                raw = ncu_csv(rep, "raw")
                m = dict(zip(raw[0], raw[2]))
                u = dict(zip(raw[0], raw[1]))
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                tot = sum(float(m[k].replace(",", "")) * scale.get(u[k], 1)
                          for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
                traffic[kname] = {"dram_bytes": tot, "alg_bytes": abytes,
                                  "source": f"profiles/{tag}/ncu_summary.md "
                                            f"({os.path.basename(rep)}, tools/prof_driver.py {key})"}
    # pipe utilisation of the compute-bound kernels (bench.py reports it beside
    # the algorithmic roofline)
    for rep in args:
        for key in ("fisher4", "fisher10", "normal", "exponential"):
            if f"prof_{key}_" in os.path.basename(rep):
                raw = ncu_csv(rep, "raw")
                m = dict(zip(raw[0], raw[2]))

                def f(k):
                    try:
                        return float(m[k].replace(",", ""))
                    except (KeyError, ValueError):
                        return None

                traffic[f"pipes_{key}"] = {
                    "fp64_pipe_active_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                    "issue_slots_busy_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
                    "alu_pct": f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                    "xu_pct": f("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                    "threads_per_warp_inst": f("smsp__thread_inst_executed_per_inst_executed.ratio"),
                    "source": f"profiles/{tag}/ncu_summary.md ({os.path.basename(rep)})"}
    if traffic:
        with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as fh:
            import json

            json.dump(traffic, fh, indent=1)
    if lcsv:
        import shutil

        shutil.copy(lcsv, os.path.join(outdir, "launches.csv"))
        with open(os.path.join(outdir, "launches.md"), "w") as fh:
            fh.write(f"# Launch list ({tag}): `ncu --metrics gpu__time_duration.sum "
                     "--clock-control none` over `bench.py --steps 4 --warmup 3 --no-cpu`\n\n")
            fh.write("Cold-cache serialised launches: compare shares, not absolutes.\n\n")
            fh.write(launches(lcsv))
    print("wrote", outdir)


if __name__ == "__main__":
    main()
