timeout 300 python tools/debug_inplace.py > gpurun_out/r02f_debug.log 2>&1
