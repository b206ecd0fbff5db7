# C5 bench value for relabel periods (measurement only; bench --relabel-every)
for r in 32 64 128 256; do
  timeout 300 python bench.py --steps 200 --warmup 20 --late-t 700 --no-e2e --no-cpu --relabel-every $r > gpurun_out/rl_$r.json 2> /dev/null
done
