"""One line per kernel launch of an `ncu --set full` report (diagnostic):
duration, DRAM and L2 traffic, L2 hit rate, SM / memory throughput,
occupancy, registers, grid, block.

usage: python tools/ncu_summary.py report.ncu-rep "<header line>" > summary.txt
"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
           "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
           "launch__block_size"]
SCALE = {"ms": 1e3, "us": 1.0, "ns": 1e-3, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3,
         "Gbyte": 1e3, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6}


def short(name):
    name = name.replace("void ", "")
    head = name.split("(")[0]
    return head.replace("f4b::", "")


def main():
    rep, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cols, units = rows[0], rows[1]
    ix = {c: i for i, c in enumerate(cols)}

    def val(r, m):
        v = float(r[ix[m]].replace(",", ""))
        return v * SCALE.get(units[ix[m]], 1.0)

    if header:
        print(header)
    print("# dram_MB = dram__bytes_read + dram__bytes_write; L2_MB = lts__t_sectors x 32 B")
    print(f"{'kernel':26s} {'dur_us':>7s} {'dram_MB':>8s} {'L2_MB':>8s} {'L2hit%':>7s} {'SM%':>6s} {'mem%':>6s} "
          f"{'occ%':>6s} {'regs':>5s} {'grid':>5s} {'blk':>4s}")
    for r in rows[2:]:
        if len(r) < len(cols):
            continue
        print(f"{short(r[ix['Kernel Name']])[:26]:26s} {val(r, 'gpu__time_duration.sum'):7.1f} "
              f"{val(r, 'dram__bytes_read.sum') + val(r, 'dram__bytes_write.sum'):8.2f} "
              f"{float(r[ix['lts__t_sectors.sum']].replace(',', '')) * 32 / 1e6:8.1f} "
              f"{val(r, 'lts__t_sector_hit_rate.pct'):7.1f} "
              f"{val(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
              f"{val(r, 'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed'):6.1f} "
              f"{val(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} "
              f"{int(val(r, 'launch__registers_per_thread')):5d} {int(val(r, 'launch__grid_size')):5d} "
              f"{int(val(r, 'launch__block_size')):4d}")


if __name__ == "__main__":
    main()
