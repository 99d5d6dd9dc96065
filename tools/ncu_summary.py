"""Summarises an ncu report (and optional launch-list CSV) into profiles/ (run in the build container).

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [gpurun_out/launches.csv] --out profiles/r01_expand
Writes <out>.json (key metrics), <out>_stalls.txt (top SASS stall sites) and, with a launch list,
<out>_launches.txt (per-kernel share of the step).
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("launches", nargs="?")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rows = ncu_csv(a.rep, "raw")
    h, units, v = rows[0], rows[1], rows[2]
    res = {"kernel": v[h.index("Kernel Name")], "report": a.rep}
    stalls = {}
    for i, name in enumerate(h):
        if name in KEYS:
            res[name] = f"{v[i]} {units[i]}".strip()
        if name.startswith("smsp__pcsamp_warps_issue_stalled") and not name.endswith("not_issued"):
            try:
                stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(float(v[i].replace(",", "")))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1
    res["stall_samples_pct"] = {k: round(100 * c / tot, 1) for k, c in sorted(stalls.items(), key=lambda x: -x[1])
                                if c > 0.005 * tot}
    with open(a.out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    src = ncu_csv(a.rep, "source", ("--print-source", "sass"))
    hdr = src[1]
    ai, si, ni = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in src[2:]:
        try:
            data.append((int(r[ni] or 0), r[si]))
        except (ValueError, IndexError):
            pass
    total = sum(d[0] for d in data) or 1
    with open(a.out + "_stalls.txt", "w") as f:
        f.write(f"top SASS stall sites ({total} samples)\n")
        for c, s in sorted(data, reverse=True)[:30]:
            f.write(f"{100 * c / total:5.1f}%  {s.strip()}\n")
    if a.launches:
        lrows = list(csv.reader(open(a.launches)))
        i0 = next(i for i, r in enumerate(lrows) if r and r[0] == "ID")
        lh = lrows[i0]
        ki, vi = lh.index("Kernel Name"), lh.index("Metric Value")
        agg = defaultdict(list)
        for r in lrows[i0 + 1:]:
            if len(r) > vi:
                agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
        tot_ns = sum(sum(x) for x in agg.values())
        with open(a.out + "_launches.txt", "w") as f:
            f.write("kernel | launches | mean us | share of all launch time (cold-cache, serialised)\n")
            for k, x in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
                f.write(f"{k} | {len(x)} | {sum(x) / len(x) / 1e3:.2f} | {100 * sum(x) / tot_ns:.2f}%\n")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
