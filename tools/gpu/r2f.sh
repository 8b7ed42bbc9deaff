ncu --set full --import-source on -k regex:k4_sort -c 1 -o gpurun_out/k4_n8 python tools/gpu/sort_probe.py 8 > gpurun_out/ncu_k4.log 2>&1
tail -3 gpurun_out/ncu_k4.log
