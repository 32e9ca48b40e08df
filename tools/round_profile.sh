#!/usr/bin/env bash
# One GPU session's evidence for profiles/ (run under gpurun from the repo root; round tag in $1,
# default r02): the launch list of the default bench (configs[3]), one ncu --set full capture per
# hot kernel (cg_stream, the LS-SPAI kernel) exported to CSV on the box (the .ncu-rep files are too
# large to travel back), and the clock64 phase profiles of the streaming kernel.  Everything
# lands in gpurun_out/; summaries are copied into profiles/ by hand (tools/ncu_summary.py works on
# the raw CSV too, tools/ncu_lines.py on the source CSV).
set -u
R=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_config3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
cap() { # name, kernel regex, bench args...
  local name=$1 rx=$2
  shift 2
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$rx -c 1 -f -o /tmp/$name \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline "$@" > $O/ncu_$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>> $O/ncu_$name.log
  ncu -i /tmp/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>> $O/ncu_$name.log
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > /tmp/${name}_source.csv 2>> $O/ncu_$name.log
  python tools/ncu_lines.py /tmp/${name}_source.csv 60 > $O/${name}_hot_lines.txt 2>&1
  gzip -c /tmp/${name}_source.csv > $O/${name}_source.csv.gz
}
cap ${R}_cg_stream_config3 cg_stream --budget 100
cap ${R}_ls_columns_config3 ls_columns --budget 10
cap ${R}_cg_stream_config2 cg_stream --workload config2 --budget 200
timeout 600 python tools/stream_prof.py 100 500000 4 16 18 > $O/${R}_stream_prof_c3.txt 2>&1
timeout 600 python tools/stream_prof.py 1000 50000 1 8 1 > $O/${R}_stream_prof_c2.txt 2>&1
du -sh $O
echo done > $O/round_profile.done
