"""Key counters of an `ncu --set full` capture (its --page raw --csv export) as text."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active % (active cycles)"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor memory (TMEM) active %"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc pipe inst %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / scheduler"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2 -> SM bytes"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
print(d.get("Kernel Name", ("", "?"))[1][:120])
for k, label in KEYS:
    if k in d:
        print(f"  {label:40s} {d[k][1]:>14s} {d[k][0]}")
st = [(float(v.replace(",", "")), h) for h, (u, v) in d.items()
      if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and v.replace(",", "").replace(".", "").isdigit()]
tot = sum(v for v, _ in st) or 1.0
print("  stall samples (top 6):")
for v, h in sorted(st, reverse=True)[:6]:
    print(f"    {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:5.1f} %")
