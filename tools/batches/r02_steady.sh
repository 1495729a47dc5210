# steady-state co-run tables (every kind scaled to a >= 2 ms solo run): OPT table and model error
set -x
KL_STEADY=1 timeout 2400 python tools/opt_table.py gpurun_out/r02_opt_table_steady.json > gpurun_out/opt_steady.log 2>&1
KL_STEADY=1 timeout 1800 python tools/model_error.py gpurun_out/r02_model_error_steady.json > gpurun_out/me_steady.log 2>&1
tail -12 gpurun_out/me_steady.log
