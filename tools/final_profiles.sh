#!/bin/bash
# Round-end evidence on the GPU box: launch list of the bench command, full
# ncu captures of the bench kernel per strategy and of the other configs
# (summarised on the box), and the bench line.  (compute-sanitizer is closed
# on this pool: correctness rests on the parity suites.)
set -x
O=gpurun_out/${1:-r2final}
mkdir -p $O
lib=paper_2006_07478_b200/lib/librs.so
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-sweep --no-check > /dev/null 2>&1
summ() {   # report kernel items name
  { python tools/summarize_ncu.py $1; echo; echo "## executed warp-instructions per child by inline call chain (tools/inline_prof.py)";
    python tools/inline_prof.py $1 $lib $2 $3 0.004 7;
    echo; echo "## warp-stall samples by inline call chain";
    COL="Warp Stall Sampling (All Samples)" python tools/inline_prof.py $1 $lib $2 1 0.004 7; } 2>&1
}
for s in signal tagged context; do
  ncu --set full --clock-control none --import-source on -k regex:k_pipeline -s 3 -c 1 -o /tmp/prof_$s \
      python bench.py --strategy $s --steps 1 --warmup 3 --no-e2e --no-cpu --no-sweep --no-check > /dev/null 2>&1
  k=k_pipelineILi3ELi20ELb0ELb1ELb0ELb0ELi0ELb0ELb0E
  [ $s = tagged ] && k=k_pipelineILi3ELi20ELb1ELb1ELb0ELb0ELi0ELb0ELb0E
  [ $s = context ] && k=k_pipelineILi3ELi20ELb0ELb1ELb1ELb0ELi0ELb0ELb0E
  summ /tmp/prof_$s.ncu-rep $k 536870912 > $O/summary_$s.txt
  ncu -i /tmp/prof_$s.ncu-rep --page raw --csv > $O/raw_$s.csv 2>/dev/null
done
# other configs (1-GPU points): variable L = 4096, Zipf, text; the short-region kernel at L = 1
for wk in "sweep_var_L4096 signal k_pipelineILi3ELi20ELb0ELb1ELb0ELb0ELi0ELb0ELb0E 536870912 0" \
          "zipf tagged k_pipelineILi3ELi20ELb1ELb1ELb0ELb0ELi0ELb0ELb0E 1071868463 0" \
          "text signal k_pipelineILi1ELi23ELb0ELb1ELb0ELb0ELi0ELb0ELb0E 4294967296 0" \
          "sweep_fixed_L1 signal k_pipelineILi3ELi20ELb0ELb1ELb0ELb0ELi0ELb0ELb1E 536870912 256"; do
  set -- $wk
  ncu --set full --clock-control none --import-source on -k regex:k_pipeline -s 3 -c 1 -o /tmp/prof_$1 \
      python tools/cfg_sweep.py --reps 1 --workload $1 --strategy $2 --flags $5 0:0:0 > /dev/null 2>&1
  summ /tmp/prof_$1.ncu-rep $3 $4 > $O/summary_$1_$2.txt
done
python bench.py > $O/bench.log 2>&1
