"""Summarise an ncu report (--page raw) into the metrics the roofline needs."""
import csv, io, subprocess, sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "l1tex__t_bytes.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum"]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        name = d[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        m = {"kernel": name[:90]}
        for w in WANT:
            if w in hdr:
                m[w] = f"{d[hdr.index(w)]} {units[hdr.index(w)]}"
        st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(d[i].replace(",", "") or 0))
              for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1
        m["stalls_top"] = ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in sorted(st, key=lambda t: -t[1])[:7])
        res.append(m)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for m in summarise(p):
            print(f"== {p}")
            for k, v in m.items():
                print(f"  {k}: {v}")
