"""One CSV row per ncu --set full capture: duration, DRAM bytes, throughput
fractions, registers, launch shape, instructions
(python tools/ncu_summary.py a.ncu-rep [b.ncu-rep ...])."""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
     "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct"]
print("kernel,duration_us,dram_read_bytes,dram_write_bytes,mem_pct_peak,sm_pct_peak,regs,grid,block,"
      "instructions,l2_hit_pct,report")
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        v = dict(zip(hdr, r))
        u = dict(zip(hdr, units))

        def num(k, scale=None):
            x = float(v.get(k, "nan").replace(",", "") or "nan")
            unit = u.get(k, "")
            if scale == "us":
                x = x / 1e3 if unit == "ns" else (x * 1e3 if unit in ("ms", "msecond") else x)
            if scale == "B":
                x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return x
        print(f"{v['Kernel Name'].split('(')[0]},{num(M[0], 'us'):.2f},{num(M[1], 'B'):.0f},{num(M[2], 'B'):.0f},"
              f"{num(M[3]):.3f},{num(M[4]):.3f},{num(M[5]):.0f},{num(M[6]):.0f},{num(M[7]):.0f},{num(M[8]):.0f},"
              f"{num(M[9]):.1f},{rep.split('/')[-1]}")
