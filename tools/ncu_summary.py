"""Summaries committed under profiles/ (read here with the ncu CLI).

  python tools/ncu_summary.py launches <launches.csv>      per-kernel share of a launch list
  python tools/ncu_summary.py report <rep.ncu-rep> [name]  key metrics + stall reasons + hot lines
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("Grid Size", "launch__grid_size"), ("Block Size", "launch__block_size"),
    ("Duration", "gpu__time_duration.sum"),
    ("DRAM read", "dram__bytes_read.sum"), ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM throughput % peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("SM throughput % peak", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("Mem throughput % peak", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("Warps active % peak", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("Threads per warp inst", "smsp__thread_inst_executed_per_inst_executed.ratio"),
    ("Issue slots busy %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("L1 hit %", "l1tex__t_sector_hit_rate.pct"), ("L2 hit %", "lts__t_sector_hit_rate.pct"),
    ("Registers/thread", "launch__registers_per_thread"),
    ("Dyn smem/block", "launch__shared_mem_per_block_dynamic"),
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
              "nsecond": 1e-6}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k[:40]:40s} {cnt[k]:8d} {v:10.3f} {100 * v / s:6.1f}%")
    print(f"{'all':40s} {sum(cnt.values()):8d} {s:10.3f}")


def report(path, name=None):
    raw = list(csv.reader(io.StringIO(ncu("-i", path, "--page", "raw", "--csv"))))
    hdr, units = raw[0], raw[1]
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        kname = d["Kernel Name"]
        if name and name not in kname:
            continue
        print(f"kernel: {kname}")
        for label, key in KEYS:
            if key in d:
                print(f"  {label:26s} {d[key]} {u.get(key, '')}")
        st = [(float(d[k]), k.replace("smsp__pcsamp_warps_issue_stalled_", ""))
              for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("not_issued") and d[k].replace(".", "", 1).isdigit()]
        tot = sum(x for x, _ in st) or 1
        print("  stall reasons (pc samples):")
        for x, k in sorted(st, reverse=True)[:8]:
            print(f"    {k:28s} {100 * x / tot:5.1f}%")
        kn = kname.split("(")[0].split()[-1].split("<")[0]
        src = ncu("-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{kn}",
                  "--print-source", "cuda,sass")
        lines, hdr2 = [], None
        for r in csv.reader(io.StringIO(src)):
            if r and r[0] == "Line No":
                hdr2 = r
                continue
            if hdr2 is None or not r or not r[0]:
                continue
            dd = dict(zip(hdr2[4:], r[4:]))
            try:
                lines.append((int(dd["Warp Stall Sampling (All Samples)"]),
                              int(dd["Instructions Executed"]), r[0], r[1].strip()[:80]))
            except (KeyError, ValueError):
                pass
        ts = sum(x[0] for x in lines) or 1
        ti = sum(x[1] for x in lines) or 1
        print("  hottest source lines (stall samples %, warp instructions %):")
        for s_, i_, ln, text in sorted(lines, reverse=True)[:15]:
            print(f"    {100 * s_ / ts:5.1f}% {100 * i_ / ti:5.1f}%  L{ln:>5}  {text}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
