# kNN stage times at C5 for pilot windows / locality-cell counts (measurement only)
run() {
  tag=$1; shift
  TSNE_NVCC_EXTRA="$*" python paper_1807_11824_b200/build.py --force > /dev/null 2>&1
  TSNE_KNN_TIMING=1 timeout 600 python measure/knn_stages.py > gpurun_out/kp_$tag.log 2>&1
}
run w4 "-DTSNE_SYM_WINDOW=4"
run w5 "-DTSNE_SYM_WINDOW=5"
TSNE_NVCC_EXTRA="-DTSNE_SYM_WINDOW=6" python paper_1807_11824_b200/build.py --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_knn_p.py -x -q > gpurun_out/kp_w6_tests.log 2>&1; echo EXIT $? >> gpurun_out/kp_w6_tests.log
python paper_1807_11824_b200/build.py --force > /dev/null 2>&1
