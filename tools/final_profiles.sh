#!/bin/bash
# Round-end evidence on the GPU box: launch list of the bench command, full
# ncu captures of the bench kernel per strategy and of the other configs
# (summarised on the box), and the bench line.
set -x
O=gpurun_out/r2final
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-sweep --no-check > /dev/null 2>&1
lib=paper_2006_07478_b200/lib/librs.so
for s in signal tagged context; do
  ncu --set full --clock-control none --import-source on -k regex:k_pipeline -s 3 -c 1 -o /tmp/prof_$s \
      python bench.py --strategy $s --steps 1 --warmup 3 --no-e2e --no-cpu --no-sweep --no-check > /dev/null 2>&1
  k=k_pipelineILi3ELi20ELb0ELb1ELb0ELb0ELi0E
  [ $s = tagged ] && k=k_pipelineILi3ELi20ELb1ELb1ELb0ELb0ELi0E
  [ $s = context ] && k=k_pipelineILi3ELi20ELb0ELb1ELb1ELb0ELi0E
  { python tools/summarize_ncu.py /tmp/prof_$s.ncu-rep; echo; echo "## hot instruction footprint (tools/hot_footprint.py)";
    python tools/hot_footprint.py /tmp/prof_$s.ncu-rep; echo;
    echo "## hot code and no-instruction stalls by function (tools/code_map.py)";
    python tools/code_map.py /tmp/prof_$s.ncu-rep $lib $k 1e-4; echo;
    echo "## executed warp-instructions per child by source line (tools/line_prof.py, top 30)";
    python tools/line_prof.py /tmp/prof_$s.ncu-rep $lib $k 536870912 30; } > $O/summary_$s.txt 2>&1
  ncu -i /tmp/prof_$s.ncu-rep --page raw --csv > $O/raw_$s.csv 2>/dev/null
done
# other configs (1-GPU points): variable L = 4096, Zipf, text
for wk in "sweep_var_L4096 signal k_pipelineILi3ELi20ELb0ELb1ELb0ELb0ELi0E" "zipf tagged k_pipelineILi3ELi20ELb1ELb1ELb0ELb0ELi0E" \
          "text signal k_pipelineILi1ELi23ELb0ELb1ELb0ELb0ELi0E"; do
  set -- $wk
  ncu --set full --clock-control none --import-source on -k regex:k_pipeline -s 3 -c 1 -o /tmp/prof_$1 \
      python tools/cfg_sweep.py --reps 1 --workload $1 --strategy $2 0:0:0 > /dev/null 2>&1
  { python tools/summarize_ncu.py /tmp/prof_$1.ncu-rep; echo; python tools/code_map.py /tmp/prof_$1.ncu-rep $lib $3 1e-4; } \
      > $O/summary_$1_$2.txt 2>&1
done
python bench.py > $O/bench.log 2>&1
{ compute-sanitizer --tool memcheck --error-exitcode 0 python tools/sanitize_cases.py 2>&1 | tail -4;
  compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_cases.py 2>&1 | tail -4; } > $O/sanitizer.txt
