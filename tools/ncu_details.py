"""Text summary of an ncu --set full report (details page): the throughput,
issue, occupancy and shared-memory lines the profiles/ summaries quote.

    python tools/ncu_details.py report.ncu-rep [--raw] > profiles/rNN_ncu_full_X.txt
"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput",
        "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "No Eligible"]
RAW = ["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
       "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = {k: i for i, k in enumerate(rows[0])}
    for r in rows[1:]:
        name = r[h["Metric Name"]]
        if name in WANT:
            print(f"{r[h['Kernel Name']].split('(')[0]} | {name} {r[h['Metric Unit']]} | {r[h['Metric Value']]}")
    if "--raw" in sys.argv:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            kn = r[hdr.index("Kernel Name")].split("(")[0]
            for m in RAW:
                if m in hdr:
                    print(f"{kn} | {m} {units[hdr.index(m)]} | {r[hdr.index(m)]}")


if __name__ == "__main__":
    main()
