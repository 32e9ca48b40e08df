"""Summarise one ncu --set full report (first kernel) into the JSON kept under profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep|REPORT_raw.csv KEY NOTE [SUMMARY.json [ITERATIONS [WORKLOAD_KEY]]]
prints the summary and merges it under KEY into the summary file (default profiles/r02_ncu_summary.json).
REPORT_raw.csv is `ncu -i REP --page raw --csv` (tools/round_profile.sh exports it on the GPU box).
ITERATIONS (CG iterations of the captured launch) adds dram_bytes_per_cg_iteration; WORKLOAD_KEY
(bench.py --workload name) lets bench.py report it as roofline.traffic, guarded by a hash of the
streaming kernel's source files taken now (capture and summary belong to the same tree).
"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SOURCES = ["paper_1606_01216_b200/csrc/cg_stream.cu", "paper_1606_01216_b200/csrc/cg_common.cuh"]

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "smsp__warps_active.avg.per_cycle_active", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__average_warp_latency_issue_stalled_barrier", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "launch__shared_mem_per_block_dynamic",
]

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    rep, key, note = sys.argv[1], sys.argv[2], sys.argv[3]
    out = sys.argv[4] if len(sys.argv) > 4 else "profiles/r02_ncu_summary.json"
    its = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    wkey = sys.argv[6] if len(sys.argv) > 6 else None
    if rep.endswith(".csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, first = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}
    summ = {"Kernel Name": first[col["Kernel Name"]]}
    for m in METRICS:
        if m in col:
            summ[m] = f"{first[col[m]]} {units[col[m]]}".strip()
    rd = float(first[col["dram__bytes_read.sum"]].replace(",", "")) * UNIT.get(units[col["dram__bytes_read.sum"]], 1)
    wr = float(first[col["dram__bytes_write.sum"]].replace(",", "")) * UNIT.get(units[col["dram__bytes_write.sum"]], 1)
    summ["dram_bytes_per_launch"] = rd + wr
    if its:
        summ["dram_bytes_per_cg_iteration"] = (rd + wr) / its
    if wkey:
        h = hashlib.sha256()
        for rel in SOURCES:
            with open(os.path.join(ROOT, rel), "rb") as f:
                h.update(f.read())
        summ["workload_key"] = wkey
        summ["source_files"] = SOURCES
        summ["source_sha16"] = h.hexdigest()[:16]
    summ["note"] = note
    try:
        with open(out) as f:
            allsum = json.load(f)
    except FileNotFoundError:
        allsum = {}
    allsum[key] = summ
    with open(out, "w") as f:
        json.dump(allsum, f, indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
