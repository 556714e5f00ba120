"""Summarise an ncu report (raw page) into one line per profiled kernel:
duration, DRAM bytes, tensor-pipe / L2 / DRAM / SM utilisation, grid, regs.
usage: python tools/ncu_summary.py report.ncu-rep [> profiles/xxx.txt]"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("dur_us", "gpu__time_duration.sum", 1e-3),
    ("dram_rd_MB", "dram__bytes_read.sum", 1.0),
    ("dram_wr_MB", "dram__bytes_write.sum", 1.0),
    ("hmma_cyc", "TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", 1.0),
    ("tc_inst%", "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", 1.0),
    ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("l2%", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("l1%", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1.0),
    ("sm%", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("grid", "launch__grid_size", 1.0),
    ("regs", "launch__registers_per_thread", 1.0),
    ("smem_KB", "launch__shared_mem_per_block_dynamic", 1.0),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    name = h.index("Kernel Name")
    print("kernel | " + " | ".join(m[0] for m in METRICS))
    for r in rows[2:]:
        vals = []
        for label, key, _ in METRICS:
            if key not in h:
                vals.append("-")
                continue
            i = h.index(key)
            v = r[i].replace(",", "")
            u = units[i]
            try:
                f = float(v)
                if key.startswith("dram__bytes"):
                    f = f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                if key == "gpu__time_duration.sum":
                    f = f * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
                if key == "launch__shared_mem_per_block_dynamic":
                    f = f * {"byte": 1 / 1024, "Kbyte": 1.0}.get(u, 1.0)
                vals.append(f"{f:.1f}")
            except ValueError:
                vals.append(v[:12])
        print(r[name].split("(")[0][:28] + " | " + " | ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
