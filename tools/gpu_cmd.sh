python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
python tools/kbench.py --configs C1,C2,C4,C3,C5 --paths BUCKETED > gpurun_out/kbench.log 2>&1
python tools/run_one.py --config C2 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/run_one.py --config C2 > /dev/null 2>&1
python tools/run_one.py --config C4 > gpurun_out/plain4.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/run_one.py --config C4 > /dev/null 2>&1
python tools/run_one.py --config C2 --iters 1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"partition|bucket_sort" -c 2 -o gpurun_out/prof_c2 python tools/run_one.py --config C2 --iters 1 > gpurun_out/ncu_full.log 2>&1
