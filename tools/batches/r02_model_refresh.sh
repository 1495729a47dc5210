# model vs hardware (C3: 28 ALL pairs x 3 ratios at paper size) and the MM x streaming sweep with
# the final kernels
timeout 1500 python tools/model_error.py gpurun_out/f2_model_error.json > gpurun_out/f2_model_error.log 2>&1; echo "me rc $?"
timeout 1500 python tools/c3_mm_stream.py gpurun_out/f2_c3_mm_stream.json > gpurun_out/f2_c3.log 2>&1; echo "c3 rc $?"
tail -12 gpurun_out/f2_model_error.log
