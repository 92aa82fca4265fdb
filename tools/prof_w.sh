# ncu capture of one k_pipeline launch of a workload/strategy/config; summary + hot-code map
# usage: bash tools/prof_w.sh WORKLOAD STRATEGY QCAP:STAGE:SCAP KERNEL_SUBSTR TAG
w=$1; s=$2; c=$3; k=$4; t=$5
mkdir -p gpurun_out/pw
ncu --set full --clock-control none --import-source on -k regex:k_pipeline -s 3 -c 1 -o gpurun_out/pw/$t \
    python tools/cfg_sweep.py --reps 1 --workload $w --strategy $s $c > /dev/null 2>&1
python tools/summarize_ncu.py gpurun_out/pw/$t.ncu-rep > gpurun_out/pw/$t.txt 2>&1
python tools/code_map.py gpurun_out/pw/$t.ncu-rep paper_2006_07478_b200/lib/librs.so $k 1e-4 >> gpurun_out/pw/$t.txt 2>&1
