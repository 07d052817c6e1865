timeout 120 tools/bin/mc_probe > gpurun_out/r02g_mc_probe.log 2>&1; echo "exit=$?" >> gpurun_out/r02g_mc_probe.log
