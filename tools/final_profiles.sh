#!/bin/bash
# Round-end evidence on the GPU box: launch list, full ncu captures of the
# bench kernel per strategy (summarised on the box), and the bench line.
set -x
mkdir -p gpurun_out/final
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-sweep > /dev/null 2>&1
for s in signal tagged context; do
  ncu --set full --clock-control none --import-source on -k regex:k_pipeline -s 3 -c 1 -o /tmp/prof_$s \
      python bench.py --strategy $s --steps 1 --warmup 3 --no-e2e --no-cpu --no-sweep > /dev/null 2>&1
  k=k_pipelineILi3ELi20ELb0ELb1ELb0E
  [ $s = tagged ] && k=k_pipelineILi3ELi20ELb1ELb1ELb0E
  [ $s = context ] && k=k_pipelineILi3ELi20ELb0ELb1ELb1E
  { python tools/summarize_ncu.py /tmp/prof_$s.ncu-rep; echo; echo "## hot instruction footprint (tools/hot_footprint.py)";
    python tools/hot_footprint.py /tmp/prof_$s.ncu-rep; echo;
    echo "## executed warp-instructions per child by source line (tools/line_prof.py, top 30)";
    python tools/line_prof.py /tmp/prof_$s.ncu-rep paper_2006_07478_b200/lib/librs.so $k 536870912 30; } > gpurun_out/final/summary_$s.txt 2>&1
  ncu -i /tmp/prof_$s.ncu-rep --page raw --csv > gpurun_out/final/raw_$s.csv 2>/dev/null
done
python bench.py > gpurun_out/final/bench.log 2>&1
