set -x
mkdir -p gpurun_out/p1
ncu --set full --clock-control none --import-source on -k regex:k_pipeline -s 3 -c 1 -o gpurun_out/p1/sig python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-sweep > /dev/null 2>&1
k=k_pipelineILi3ELi20ELb0ELb1ELb0E
{ python tools/summarize_ncu.py gpurun_out/p1/sig.ncu-rep; echo; python tools/hot_footprint.py gpurun_out/p1/sig.ncu-rep; echo; python tools/line_prof.py gpurun_out/p1/sig.ncu-rep paper_2006_07478_b200/lib/librs.so $k 536870912 40; } > gpurun_out/p1/summary_sig.txt 2>&1
