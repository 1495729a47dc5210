# MM plain grid: first-tile L2 prefetch (product) vs none (-DKL_NO_FIRST_PREFETCH)
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "mm" > gpurun_out/ab15_tests.log 2>&1; echo rc=$? >> gpurun_out/ab15_tests.log
for r in 1 2 3; do
  timeout 200 python tools/mm_probe.py 8192x2048x2048 >> gpurun_out/ab15_prod.txt 2>&1
  KL_LIB_PATH=variants/libkl_nopf.so timeout 200 python tools/mm_probe.py 8192x2048x2048 >> gpurun_out/ab15_nopf.txt 2>&1
done
