# ncu captures of one k_pipeline launch for the given libraries on a workload
# usage: bash tools/prof_var.sh WORKLOAD LIBTAG...
w=$1; shift
mkdir -p gpurun_out/pv
for L in "$@"; do
  if [ $L = cur ]; then unset RS_LIB; else export RS_LIB=$PWD/paper_2006_07478_b200/lib/librs_$L.so; fi
  ncu --set full --clock-control none --import-source on -k regex:k_pipeline -s 3 -c 1 -o gpurun_out/pv/${w}_$L \
      python tools/cfg_sweep.py --reps 1 --workload $w 0:0:0 > /dev/null 2>&1
  python tools/summarize_ncu.py gpurun_out/pv/${w}_$L.ncu-rep > gpurun_out/pv/${w}_$L.txt 2>&1
  python tools/hot_footprint.py gpurun_out/pv/${w}_$L.ncu-rep >> gpurun_out/pv/${w}_$L.txt 2>&1
done
