"""Markdown summary of an ncu report: key metrics per launch + top stall lines."""
import csv, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def main(rep, title):
    hdr, units, data = raw(rep)
    print(f"## {title}\n\nreport: `{rep.split('/')[-1]}` (ncu --set full --clock-control none)\n")
    for r in data:
        print(f"**{r[hdr.index('Kernel Name')][:110]}**\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {k} | {r[i]} | {units[i]} |")
        print()
    lines = subprocess.run([sys.executable, "scripts/ncu_lines.py", rep, "15"], capture_output=True,
                           text=True).stdout
    print("Top source lines by warp-stall samples:\n\n```\n" + lines + "```\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
