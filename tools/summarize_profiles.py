"""Write the committed profile evidence for one profiling pass
(tools/profile_round.sh output in gpurun_out/) into profiles/:

  <tag>_c<cfg>_launches.csv          every launch of one timed V-cycle: kernel, grid,
                                     duration, DRAM bytes (cold-cache, serialised:
                                     compare shares, not absolutes)
  <tag>_c<cfg>_launch_summary.txt    per kernel x grid: launches, time, share, DRAM GB/s
  <tag>_c<cfg>_<kernel>_L0_ncu_full.csv   key metrics + stall reasons of the top
                                     kernel's level-0 launch (ncu --set full)

    python tools/summarize_profiles.py <tag> <cfg> [kernel]
"""
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_l1tex2xbar_write_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]


def main(tag, cfg, kernel="k_scgs_fwd"):
    out = os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    src = os.path.join(out, f"{tag}_c{cfg}_launches.csv")
    rows = list(csv.reader(open(src)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi, gi, mi, idi = (h.index(c) for c in ("Kernel Name", "Metric Value", "Grid Size", "Metric Name", "ID"))
    per = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        d = per.setdefault(r[idi], {"kernel": r[ki].split("(")[0].replace("void ", ""), "grid": r[gi]})
        d[r[mi]] = r[vi]
    with open(os.path.join(prof, f"{tag}_c{cfg}_launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "duration_ns", "dram_read_bytes", "dram_write_bytes"])
        for k in sorted(per, key=int):
            d = per[k]
            w.writerow([k, d["kernel"], d["grid"], d.get("gpu__time_duration.sum"), d.get("dram__bytes_read.sum"),
                        d.get("dram__bytes_write.sum")])
    summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_bw.py"), src, "40"],
                          capture_output=True, text=True).stdout
    with open(os.path.join(prof, f"{tag}_c{cfg}_launch_summary.txt"), "w") as f:
        f.write(f"# ncu launch list, one timed V-cycle of bench.py --config {cfg} (--profile-from-start off)\n")
        f.write("# kernel grid | launches | total | per launch | share | DRAM GB/s (bytes/duration)\n")
        f.write(summ)
    full_summary(tag, os.path.join(out, f"{tag}_c{cfg}_top"), os.path.join(prof, f"{tag}_c{cfg}_{kernel}_L0_ncu_full.csv"))
    if os.path.exists(os.path.join(out, f"{tag}_back_raw.csv")):
        full_summary(tag, os.path.join(out, f"{tag}_back"), os.path.join(prof, f"{tag}_c{cfg}_k_scgs_back_L0_ncu_full.csv"))
    print(open(os.path.join(prof, f"{tag}_c{cfg}_launch_summary.txt")).read())


def full_summary(tag, stem, dst):
    """key metrics + stall reasons of one ncu --set full capture: <stem>.ncu-rep,
    or its raw page already exported on the GPU box as <stem>_raw.csv"""
    if os.path.exists(stem + "_raw.csv"):
        raw = open(stem + "_raw.csv").read()
    else:
        raw = subprocess.run(["ncu", "-i", stem + ".ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, units, r = rr[0], rr[1], rr[2]
    with open(dst, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["metric", "unit", "value"])
        w.writerow(["Kernel Name", "", r[h.index("Kernel Name")]])
        for k in KEYS:
            if k in h:
                w.writerow([k, units[h.index(k)], r[h.index(k)]])
        st = [(float(r[i].replace(",", "")), h[i]) for i in range(len(h))
              if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued") and r[i]]
        tot = sum(v for v, _ in st) or 1.0
        for v, k in sorted(st, reverse=True)[:10]:
            w.writerow([k.replace("smsp__pcsamp_warps_issue_stalled_", "stall_"), "% of samples",
                        f"{100 * v / tot:.1f}"])


if __name__ == "__main__":
    main(*sys.argv[1:])
