#!/usr/bin/env bash
# One GPU session's evidence for profiles/ (run under gpurun from the repo root):
# bench lines (ours + the reference arm), the configs[1] launch list, one ncu --set full
# capture per hot kernel (cg_cluster_v2 on configs[1], cg_stream on configs[3]) and the
# configs[2] AIRGA sequence.  Everything lands in gpurun_out/; summaries are copied into
# profiles/ by hand (tools/ncu_summary.py, tools/ncu_lines.py).
set -u
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 600 python bench.py > $O/bench_c1.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1
timeout 600 python bench.py --workload config3 --steps 5 --warmup 3 > $O/bench_c3.log 2>&1
timeout 600 python bench.py --workload config2 --steps 10 --warmup 3 > $O/bench_c2.log 2>&1
timeout 900 python bench.py --workload config4 --steps 2 --warmup 3 > $O/bench_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cg_cluster_v2 -c 1 -f -o $O/cluster_c1 \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_cluster.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cg_stream -c 1 -f -o $O/stream_c3 \
  python bench.py --workload config3 --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_stream.log 2>&1
timeout 900 python tools/airga_sequence.py --ref-budget 20 --out $O/airga_sequence.json > $O/airga_seq.log 2>&1
echo done > $O/round_profile.done
