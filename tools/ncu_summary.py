"""Summarise ncu reports for profiles/: per launch -- duration, DRAM bytes
read+written, DRAM / L2 / SM throughput, tensor-pipe activity, registers,
occupancy -- plus the top stall lines of the source page.
usage: python tools/ncu_summary.py REPORT.ncu-rep [--stalls N]"""
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "sm__warps_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")][:60]}
        for m in RAW:
            if m in hdr:
                i = hdr.index(m)
                d[m] = (r[i], units[i])
        # tensor pipe activity (tcgen05 UTC*MMA shows up in the tensor pipe counters)
        for h in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active"):
            if h in hdr and h not in d:
                i = hdr.index(h)
                d[h] = (r[i], units[i])
        res.append(d)
    return res


def stalls(rep, n):
    """Top stall lines of the FIRST kernel on the source page (the page holds one
    header + body block per profiled kernel)."""
    out = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    key = "Warp Stall Sampling (All Samples)"
    start = next((k for k, r in enumerate(rows) if key in r), None)
    if start is None:
        return []
    hdr = rows[start]
    i = hdr.index(key)
    body = []
    for r in rows[start + 1:]:
        if key in r or (r and r[0] == "Kernel Name"):
            break  # the next kernel's block
        if len(r) > i and r[i].isdigit():
            body.append(r)
    tot = sum(int(r[i]) for r in body) or 1
    top = sorted(body, key=lambda r: -int(r[i]))[:n]
    return [(int(r[i]) / tot, r[1].strip()) for r in top]


def main():
    rep = sys.argv[1]
    n = int(sys.argv[sys.argv.index("--stalls") + 1]) if "--stalls" in sys.argv else 8
    print(f"# ncu summary of {rep.split('/')[-1]}")
    for k, d in enumerate(raw(rep)):
        print(f"\n## launch {k}: {d.pop('kernel')}")
        for m, (v, u) in d.items():
            print(f"  {m:70s} {v} {u}")
    st = stalls(rep, n)
    if st:
        print("\n## top stall sites (first launch, share of warp-stall samples)")
        for frac, src in st:
            print(f"  {frac:6.1%}  {src[:110]}")


if __name__ == "__main__":
    main()
