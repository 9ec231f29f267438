"""Summarise an ncu --set full capture (raw page CSV) into the metric table
kept under profiles/: python profiles/ncu_summary.py raw.csv > summary.csv"""
import csv
import sys

WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def main(path):
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    w = csv.writer(sys.stdout)
    w.writerow(["kernel", "metric", "unit", "value"])
    for v in rows[2:]:
        name = v[h.index("Kernel Name")][:60] if "Kernel Name" in h else "?"
        for m in WANT[1:]:
            if m in h:
                i = h.index(m)
                w.writerow([name, m, u[i], v[i]])


if __name__ == "__main__":
    main(sys.argv[1])
