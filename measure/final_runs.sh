# Round-end evidence (run from the repo root on the GPU box): the GPU suite and
# smoke(), bench lines of every configuration (C5 = the headline), the reference
# arm, the ncu launch list of the default bench command, and full ncu captures of
# the iteration kernels at C5.
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/fin_gputest.log 2>&1; echo "EXIT $?" >> gpurun_out/fin_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1
for c in C5 C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 20 --late-t 700 > gpurun_out/fin_bench_$c.json 2> gpurun_out/fin_bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_reference.json 2> gpurun_out/fin_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/fin_launches_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --nvtx --nvtx-include "profile/" --csv --log-file gpurun_out/fin_launches_profile.csv python bench.py --steps 20 --warmup 20 --no-e2e --no-cpu > gpurun_out/fin_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_attract_tma|k_traverse|k_radix_build|k_quad_emit" --launch-skip 60 --launch-count 5 -o gpurun_out/fin_full python bench.py --steps 20 --warmup 20 --no-e2e --no-cpu > gpurun_out/fin_full.log 2>&1
