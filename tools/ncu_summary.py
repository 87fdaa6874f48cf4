"""Summarise an ncu report: key metrics + top stall sites (for profiles/)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, top=25, kernel=None):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    pick = [r for r in rows[2:] if kernel is None or kernel in r[ki]]
    vals = pick[0]
    print(f"# {rep}")
    print(f"kernel: {vals[hdr.index('Kernel Name')][:120]}")
    for k in KEYS:
        for i, h in enumerate(hdr):
            if h.endswith(k):
                print(f"{k} = {vals[i]} {units[i]}")
    if kernel is not None:
        return  # per-kernel source pages of multi-kernel reports: capture separately
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv"]))))
    h = src[1]
    isrc, iall, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Instructions Executed")
    # multi-kernel reports: the source page repeats a title + header per
    # kernel; keep the first kernel's rows
    data = []
    for r in src[2:]:
        if len(r) <= iall or not r[iall].strip().isdigit():
            if data:
                break
            continue
        data.append(r)
    tot = sum(int(r[iall] or 0) for r in data)
    print(f"stall samples total: {tot}")
    for k, r in sorted(enumerate(data), key=lambda kr: -int(kr[1][iall] or 0))[:top]:
        print(f"  [{k:5d}] {int(r[iall]):8d} ({100*int(r[iall])/max(tot,1):5.1f}%) "
              f"exec={r[iex]:>10}  {r[isrc].strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25,
         sys.argv[3] if len(sys.argv) > 3 else None)
