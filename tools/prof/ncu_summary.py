"""Markdown summary of an ncu report (--page raw): one column per kernel
launch for the metrics the roofline discussion uses."""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "DRAM read % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX throughput"),
    ("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
     "L1->XBAR request port busy"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit rate"),
    ("lts__t_requests_srcunit_l1_op_read.sum", "L2 read requests from L1"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput"),
    ("lts__t_tag_requests.max.pct_of_peak_sustained_elapsed", "L2 tag requests, busiest slice"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (occupancy)"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue active"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    names = [r[col["Kernel Name"]][:48] for r in data]
    print("| metric | " + " | ".join(names) + " |")
    print("|---" * (len(names) + 1) + "|")
    for key, label in METRICS:
        if key not in col:
            continue
        vals = [r[col[key]] for r in data]
        print(f"| {label} [{units[col[key]]}] | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
