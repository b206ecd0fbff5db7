run() {
  tag=$1; shift
  TSNE_NVCC_EXTRA="$*" python paper_1807_11824_b200/build.py --force > /dev/null 2>&1 || { echo BUILD FAIL $tag; return; }
  timeout 240 python bench.py --steps 200 --warmup 20 --late-t 700 --no-e2e --no-cpu > gpurun_out/sw2_${tag}.json 2> gpurun_out/sw2_${tag}.err
}
run g100 "-DTSNE_AT_GRID_SHARED=100"
run g110 "-DTSNE_AT_GRID_SHARED=110"
run g120 ""
run g132 "-DTSNE_AT_GRID_SHARED=132"
run g148 "-DTSNE_AT_GRID_SHARED=148"
python paper_1807_11824_b200/build.py --force > /dev/null 2>&1
