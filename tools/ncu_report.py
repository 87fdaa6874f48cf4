"""Text summary of every launch in an ncu report (for profiles/): key
metrics per launch and the top stall sites of each launch's source page.
usage: ncu_report.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "L1 % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_size", "cluster"),
]


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, top=12):
    rows = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    print(f"# {rep}")
    for li, vals in enumerate(rows[2:]):
        print(f"\n## launch {li}: {vals[ki][:150]}")
        for key, label in KEYS:
            for i, h in enumerate(hdr):
                if h == key:
                    print(f"  {label:16s} {vals[i]} {units[i]}")
        src = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--launch-skip",
                                                   str(li), "--launch-count", "1"]))))
        if len(src) < 3:
            continue
        h = src[1]
        try:
            isrc, iall, iex = (h.index("Source"), h.index("Warp Stall Sampling (All Samples)"),
                               h.index("Instructions Executed"))
        except ValueError:
            continue
        data = []
        for r in src[2:]:
            if len(r) <= max(isrc, iall, iex) or not r[iall].strip().isdigit():
                if data:
                    break
                continue
            data.append(r)
        tot = sum(int(r[iall] or 0) for r in data)
        print(f"  stall samples: {tot}; top sites:")
        for r in sorted(data, key=lambda r: -int(r[iall] or 0))[:top]:
            print(f"    {int(r[iall]):7d} ({100 * int(r[iall]) / max(tot, 1):5.1f}%) "
                  f"exec={r[iex]:>9}  {r[isrc].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
