"""Key metrics of every kernel in an ncu report (ncu -i <rep> --page raw --csv): duration, DRAM
bytes, throughput percentages, pipe utilisation, SM balance."""
import csv
import io
import subprocess
import sys

WANT = [("gpu__time_duration.sum", "dur"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
        ("lts__t_sector_hit_rate.pct", "l2hit%"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%"),
        ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
        ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc%"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
        ("sm__cycles_active.avg", "cyc_avg"), ("sm__cycles_active.max", "cyc_max"),
        ("launch__registers_per_thread", "regs"), ("sm__cycles_elapsed.avg.per_second", "clk")]
rep = sys.argv[1]
if rep.endswith(".csv"):  # an already exported raw page
    out = open(rep).read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
for r in rows[2:]:
    name = r[idx["Kernel Name"]].split("(")[0]
    vals = []
    for m, short in WANT:
        if m in idx and r[idx[m]] not in ("", "n/a"):
            vals.append(f"{short}={r[idx[m]]}{units[idx[m]] if units[idx[m]] not in ('', '%') else ''}")
    print(name, "|", " ".join(vals))
