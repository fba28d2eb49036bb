"""Summarise ncu output into profiles/ (run here, on the CPU box).

    python tools/summarize_ncu.py launches gpurun_out/launches.csv  > profiles/<name>_launches.md
    python tools/summarize_ncu.py report   gpurun_out/prof.ncu-rep   > profiles/<name>_<kernel>.md
    python tools/summarize_ncu.py traffic  gpurun_out/prof.ncu-rep cfg2 > profiles/accumulate_traffic.json

`launches`: one timed step of the launch list (the last complete build+query
sequence), with each kernel's share of the step (cold-cache, serialised by ncu:
compare shares, not absolutes).  `report`: the headline metrics of a
--set full capture.  `traffic`: dram bytes per launch for bench.py's roofline.
"""
import collections
import csv
import io
import json
import subprocess
import sys


def short(name):
    n = name.split("(")[0]
    n = n.replace("dgsm::<unnamed>::", "").replace("void ", "")
    return n[:60]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    seq = [(int(r[ii]), short(r[ki]), float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi]
    # steps start with k_init_stats; take the last step that contains a k_query
    starts = [j for j, (_, n, _) in enumerate(seq) if n.startswith("k_init_stats")]
    best = None
    for a, b in zip(starts, starts[1:] + [len(seq)]):
        names = [n for _, n, _ in seq[a:b]]
        if any(n.startswith("k_query") for n in names):
            best = (a, b)
    a, b = best
    step = seq[a:b]
    q = next(j for j, s in enumerate(step) if s[1].startswith("k_query"))
    step = step[:q + 1]
    step = [s for s in step if not s[1].startswith("array") and "elementwise" not in s[1]]
    tot = sum(v for _, _, v in step)
    agg = collections.OrderedDict()
    for _, n, v in step:
        key = n.split("<")[0]
        agg.setdefault(key, [0, 0.0])
        agg[key][0] += 1
        agg[key][1] += v
    print(f"# ncu launch list — one step ({len(step)} kernel launches, sum {tot / 1e3:.1f} us)\n")
    print(f"source: `{path}` (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised)\n")
    print("| kernel | launches | time (us) | share |")
    print("|---|---|---|---|")
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {c} | {v / 1e3:.1f} | {100 * v / tot:.1f} % |")
    print("\n| # | kernel | us |\n|---|---|---|")
    for i, n, v in step:
        print(f"| {i} | {n} | {v / 1e3:.1f} |")


METRICS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "smsp__thread_inst_executed_per_inst_executed.ratio",
]


def raw(path):
    out = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {h[i]: (v[i], u[i]) for i in range(len(h))}
        res.append(d)
    return res


def report(path):
    for d in raw(path):
        name = short(d.get("Kernel Name", ("?", ""))[0])
        print(f"# ncu --set full: `{name}`\n\nsource: `{path}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for m in METRICS:
            if m in d:
                print(f"| {m} | {d[m][0]} | {d[m][1]} |")
        stalls = [(k, d[k][0]) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued")]
        stalls = sorted(((k, float(v or 0)) for k, v in stalls), key=lambda kv: -kv[1])[:8]
        tot = sum(float(d[k][0] or 0) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued"))
        print("\n| top stall reasons (pc samples) | share |\n|---|---|")
        for k, v in stalls:
            print(f"| {k.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {100 * v / max(tot, 1):.1f} % |")
        print()


def traffic(path, cfg, scale=1.0, kernel="accumulate", index=0):
    """DRAM bytes of the index-th captured launch of `kernel` (json on stdout)."""
    hits = [d for d in raw(path) if kernel in d.get("Kernel Name", ("", ""))[0]]
    for d in hits[index:index + 1]:
        def mb(k):
            v, u = d[k]
            f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
            return float(v) * f
        print(json.dumps({"config": cfg, "scale": scale, "kernel": f"k_{kernel}",
                          "dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
                          "dram_read": mb("dram__bytes_read.sum"), "dram_write": mb("dram__bytes_write.sum"),
                          "source": path}, indent=1))
        return


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "launches":
        launches(path)
    elif mode == "report":
        report(path)
    else:  # traffic <rep> <cfg> [kernel] [index]
        traffic(path, sys.argv[3] if len(sys.argv) > 3 else "cfg2", 1.0,
                sys.argv[4] if len(sys.argv) > 4 else "accumulate", int(sys.argv[5]) if len(sys.argv) > 5 else 0)
