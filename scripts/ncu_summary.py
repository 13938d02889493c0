"""Summarise an ncu report: key SOL metrics + top stall lines (SASS) per kernel."""
import csv
import io
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep, top=12):
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr = raw[0]
    units = dict(zip(hdr, raw[1]))
    keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        for k in keys:
            if k in d:
                print(f"  {k}: {d[k][:90]} {units.get(k, '')}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    i = [j for j, x in enumerate(src) if x and x[0] == "Address"][0]
    h = src[i]
    rows = src[i + 1:]
    S = h.index("Warp Stall Sampling (All Samples)")

    def num(x):                  # the source page repeats header rows per kernel: skip non-numbers
        try:
            return int(x[S] or 0) if len(x) > S else 0
        except ValueError:
            return 0
    tot = sum(num(x) for x in rows)
    print(f"  stall samples: {tot}")
    try:
        for x in sorted(rows, key=lambda x: -num(x))[:top]:
            print(f"    {x[S]:>6} {x[1][:100]}")
    except BrokenPipeError:
        pass


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
