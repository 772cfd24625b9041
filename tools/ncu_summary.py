"""Key metrics of an ncu --set full report (one row per profiled launch)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_active.avg", "smsp__cycles_active.avg", "launch__grid_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        res.append((d, u))
    return res


if __name__ == "__main__":
    for path in sys.argv[1:]:
        for d, u in rows(path):
            print(path.split("/")[-1], d.get("Kernel Name", "")[:60])
            for k in KEYS:
                if k in d:
                    print(f"   {k:75s} {d[k]} {u.get(k, '')}")
