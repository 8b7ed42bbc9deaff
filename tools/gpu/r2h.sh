for n in 5 11; do
ncu --set full --import-source on -k regex:k3_search -s 1 -c 1 -o gpurun_out/k3_r2_n$n python tools/gpu/k3_probe.py $n 2 > gpurun_out/ncu_k3_n$n.log 2>&1; tail -1 gpurun_out/ncu_k3_n$n.log
done
