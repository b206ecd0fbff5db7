set -x
run() {
  tag=$1; shift
  TSNE_NVCC_EXTRA="$*" python paper_1807_11824_b200/build.py --force > gpurun_out/sw_${tag}_build.log 2>&1 || { echo BUILD FAIL $tag; return; }
  timeout 240 python bench.py --steps 200 --warmup 20 --late-t 700 --no-e2e --no-cpu > gpurun_out/sw_${tag}.json 2> gpurun_out/sw_${tag}.err
}
run g120 ""
run g148 "-DTSNE_AT_GRID_SHARED=148"
run g132 "-DTSNE_AT_GRID_SHARED=132"
run g100 "-DTSNE_AT_GRID_SHARED=100"
run g80 "-DTSNE_AT_GRID_SHARED=80"
run half148 "-DTSNE_AT_GRID_SHARED=148 -DTSNE_AT_WARPS=14 -DTSNE_AT_STAGES=2 -DTSNE_AT_SMEM_LIMIT=113000"
run half100 "-DTSNE_AT_GRID_SHARED=100 -DTSNE_AT_WARPS=14 -DTSNE_AT_STAGES=2 -DTSNE_AT_SMEM_LIMIT=113000"
