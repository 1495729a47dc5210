set -x
timeout 1500 python tools/model_error.py gpurun_out/r02_model_error.json > gpurun_out/model_error.log 2>&1
timeout 1500 python tools/opt_table.py gpurun_out/r02_opt_table.json > gpurun_out/opt_table.log 2>&1
tail -12 gpurun_out/model_error.log
