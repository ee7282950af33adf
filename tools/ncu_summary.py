"""Summarise ncu captures into profiles/ (tracked).

  traffic   --csv from `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
            dram__bytes_write.sum -k regex:epsm_scan` over one launch per (sigma, m) of the
            bench sweep  ->  profiles/traffic.json (DRAM bytes per launch, bench launch mix)
  launches  --csv launch list (gpu__time_duration.sum) of the bench command -> summary text
  full      .ncu-rep of one launch (--set full) -> key metrics text
"""
import csv
import io
import json
import os
import subprocess
import sys

SIGMAS = (2, 4, 8, 16, 32, 64, 128, 256)
MS = (2, 4, 8, 16, 32)


def read_csv(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    return list(csv.DictReader(io.StringIO("".join(lines))))


def traffic(path, out_json, out_txt):
    rows = read_csv(path)
    per = {}
    for r in rows:
        if "epsm_scan" not in r["Kernel Name"] and "epsm_eqidx" not in r["Kernel Name"]:
            continue
        per.setdefault(r["ID"], {"kernel": r["Kernel Name"]})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    allk = [per[k] for k in sorted(per, key=int)]
    # keep the last len(SIGMAS) * len(MS) scans and the index builds among them (the capture
    # may hold earlier passes: the count pass, warm-up steps)
    nscan = 0
    for i in range(len(allk) - 1, -1, -1):
        if "epsm_scan" in allk[i]["kernel"]:
            nscan += 1
            if nscan == len(SIGMAS) * len(MS):
                while i > 0 and "epsm_eqidx" in allk[i - 1]["kernel"]:
                    i -= 1
                allk = allk[i:]
                break
    lines = ["sigma m  time_us  dram_read_MB  dram_write_MB   (m = 0: equality-mask index build)"]
    tot = 0.0
    launches = []
    i = 0
    for l in allk:
        rd = l["dram__bytes_read.sum"]
        wr = l["dram__bytes_write.sum"]
        s = SIGMAS[min(i // len(MS), len(SIGMAS) - 1)]
        if "epsm_eqidx" in l["kernel"]:
            lines.append("%5d %2d %8.1f %13.1f %14.1f" % (s, 0, l["gpu__time_duration.sum"] / 1e3, rd / 1e6, wr / 1e6))
            continue
        launches.append(l)
        tot += rd + wr
        m = MS[i % len(MS)]
        lines.append("%5d %2d %8.1f %13.1f %14.1f" % (s, m, l["gpu__time_duration.sum"] / 1e3, rd / 1e6, wr / 1e6))
        i += 1
    avg = tot / len(launches)
    with open(out_json, "w") as f:
        json.dump({"dram_bytes_per_launch": int(avg), "launches": len(launches),
                   "source": os.path.basename(path),
                   "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, "
                          "one search per (sigma, m) of the bench sweep (bench.py --patterns 1), "
                          "averaged with equal weight per (sigma, m) as in the bench"}, f, indent=1)
    with open(out_txt, "w") as f:
        f.write("\n".join(lines) + f"\naverage DRAM bytes per launch: {avg:.0f}\n")
    print(open(out_txt).read())


def launches(path, out_txt):
    rows = read_csv(path)
    per = []
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            per.append((r["Kernel Name"], float(r["Metric Value"].replace(",", ""))))
    mine = ("epsm_scan", "epsm_eqidx")
    ours = [t for k, t in per if "epsm_scan" in k]
    # the timed region of bench.py launches only epsm kernels: its share is taken over the
    # launches after the last non-epsm kernel (setup: text generation, pattern extraction)
    last_other = max((i for i, (k, _) in enumerate(per) if not any(x in k for x in mine)), default=-1)
    tail = per[last_other + 1:]
    with open(out_txt, "w") as f:
        f.write(f"launches captured: {len(per)} ({len(ours)} epsm_scan_kernel)\n")
        if ours:
            f.write(f"epsm_scan_kernel: sum {sum(ours)/1e3:.1f} us, mean {sum(ours)/len(ours)/1e3:.2f} us, "
                    f"min {min(ours)/1e3:.2f} us, max {max(ours)/1e3:.2f} us\n")
        tt = sum(t for _, t in tail) or 1.0
        share = sum(t for k, t in tail if "epsm_scan" in k) / tt
        ishare = sum(t for k, t in tail if "epsm_eqidx" in k) / tt
        f.write(f"launches after the last setup kernel: {len(tail)}; epsm_scan_kernel share of their "
                f"device time: {100 * share:.1f}%, epsm_eqidx_kernel (index builds) {100 * ishare:.1f}%\n")
        f.write("(ncu launch times are cold-cache and serialised: compare shares, not absolutes)\n")
    print(open(out_txt).read())


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct"]


def full(path, out_txt):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    lines = [f"ncu --set full capture: {os.path.basename(path)}", f"kernel: {v[h.index('Kernel Name')]}"]
    for k in KEYS:
        if k in h:
            i = h.index(k)
            lines.append(f"{k} = {v[i]} {u[i]}")
    stalls = [(float(v[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")) for i, n in enumerate(h)
              if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued") and v[i]]
    tot = sum(x for x, _ in stalls) or 1
    lines.append("warp stall sampling: " + ", ".join(f"{n} {100*x/tot:.1f}%" for x, n in sorted(stalls, reverse=True)[:8]))
    with open(out_txt, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(open(out_txt).read())


if __name__ == "__main__":
    kind = sys.argv[1]
    if kind == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    elif kind == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3])
