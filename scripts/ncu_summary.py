"""Summarise .ncu-rep captures (ncu --set full) into a markdown table of the
metrics that explain an HBM/L2-bound SpMV: time, DRAM bytes and throughput,
L1/L2 request-path utilisation, hit rates, occupancy, stall mix."""
import csv
import subprocess
import sys

METRICS = [
    ("duration (ms)", "gpu__time_duration.sum"),
    ("DRAM read (GB)", "dram__bytes_read.sum"),
    ("DRAM write (GB)", "dram__bytes_write.sum"),
    ("DRAM throughput % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L1TEX throughput %", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("L1->XBAR request port busy %", "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("L1 sector hit rate %", "l1tex__t_sector_hit_rate.pct"),
    ("L2 requests from L1 (read)", "lts__t_requests_srcunit_tex_op_read.sum"),
    ("L2 throughput avg %", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 tag requests max-slice %", "lts__t_tag_requests.max.pct_of_peak_sustained_elapsed"),
    ("L2 sector hit rate %", "lts__t_sector_hit_rate.pct"),
    ("warps active % (occupancy)", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("warp instructions", "smsp__inst_executed.sum"),
    ("stall long scoreboard / issue", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
    ("stall short scoreboard / issue", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"),
    ("registers / thread", "launch__registers_per_thread"),
    ("dynamic smem / CTA", "launch__shared_mem_per_block_dynamic"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def main(paths):
    cols = []
    for p in paths:
        recs, units = load(p)
        cols.append((p, recs[0], units))
    print("| metric | " + " | ".join(p.split("/")[-1] for p, _, _ in cols) + " |")
    print("|---|" + "---|" * len(cols))
    print("| kernel | " + " | ".join(r.get("Kernel Name", "?")[:60] for _, r, _ in cols) + " |")
    for label, key in METRICS:
        vals = [r.get(key, "?") for _, r, _ in cols]
        unit = cols[0][2].get(key, "")
        print(f"| {label} [{unit}] | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1:])
