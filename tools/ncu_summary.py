"""Summarise ncu captures for profiles/: per-kernel key metrics from a --set full report and the
per-launch device times from a --metrics gpu__time_duration.sum launch list.

python tools/ncu_summary.py <report.ncu-rep> <launches.csv> <out_prefix>
writes <out_prefix>_ncu_summary.md and updates profiles/ncu_traffic.json (DRAM bytes per launch)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = OrderedDict([
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA (fp32) pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_fp64.sum", "fp64 pipe instr"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
])


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append((d.get("Kernel Name", "?"), {k: (d.get(k), units[hdr.index(k)] if k in hdr else "") for k in WANT}))
    return res


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((d["Kernel Name"], float(d["Metric Value"])))
    return out


def short(name):
    s = name.split("(")[0].replace("void ", "").strip()
    for ns in ("gsicp::<unnamed>::", "gsicp::(anonymous namespace)::", "(anonymous namespace)::", "gsicp::"):
        s = s.replace(ns, "")
    return s


def main():
    rep, launches, prefix = sys.argv[1], sys.argv[2], sys.argv[3]
    lines = [f"# ncu summary ({os.path.basename(prefix)})", "",
             f"Report: `{os.path.basename(rep)}` (ncu --set full, --clock-control none; cold-cache replays), "
             f"launch list: `{os.path.basename(launches)}` (gpu__time_duration.sum, serialised).", ""]
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    seen = set()
    for name, m in raw_metrics(rep):
        s = short(name)
        if s in seen:
            continue
        seen.add(s)
        lines.append(f"## {s}")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for k, label in WANT.items():
            v, u = m[k]
            lines.append(f"| {label} (`{k}`) | {v} {u} |")
        try:
            rd = float(m["dram__bytes_read.sum"][0].replace(",", ""))
            wr = float(m["dram__bytes_write.sum"][0].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(m["dram__bytes_read.sum"][1], 1)
            wr *= scale.get(m["dram__bytes_write.sum"][1], 1)
            key = s.split("<")[0].split("::")[-1]
            traffic[key] = rd + wr
            lines.append(f"| DRAM bytes per launch (read+write) | {rd + wr:.0f} |")
        except (ValueError, AttributeError):
            pass
        lines.append("")
    # share of the step from the launch list (last complete step)
    ll = launch_list(launches)
    agg = defaultdict(float)
    cnt = defaultdict(int)
    for n, t in ll:
        agg[short(n)] += t
        cnt[short(n)] += 1
    tot = sum(agg.values())
    lines += ["## Launch list (all launches of the profiled run)", "", "| kernel | launches | total ns | share |",
              "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {cnt[k]} | {v:.0f} | {100 * v / tot:.1f}% |")
    open(prefix + "_ncu_summary.md", "w").write("\n".join(lines) + "\n")
    sys.path.insert(0, ROOT)
    from bench import csrc_sha

    traffic["_csrc_sha"] = csrc_sha()
    traffic["_capture"] = os.path.basename(rep)
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
