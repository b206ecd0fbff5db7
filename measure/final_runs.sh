# Bench lines of every configuration (C5 = the headline) and ncu evidence of the
# iteration kernels at C5 (run from the repo root on the GPU box).
set -x
for c in C5 C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 20 --late-t 700 > gpurun_out/fin_bench_$c.json 2> gpurun_out/fin_bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --nvtx --nvtx-include "profile/" --csv --log-file gpurun_out/fin_launches_profile.csv python bench.py --steps 20 --warmup 20 --no-e2e --no-cpu > gpurun_out/fin_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_attract_tma|k_traverse|k_radix_build|k_quad_emit" --launch-skip 60 --launch-count 5 -o gpurun_out/fin_full python bench.py --steps 20 --warmup 20 --no-e2e --no-cpu > gpurun_out/fin_full.log 2>&1
