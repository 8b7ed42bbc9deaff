ncu --set full --import-source on -k regex:k3_search -s 1 -c 1 -o /tmp/k3_n5 python tools/gpu/k3_probe.py 5 2 > /tmp/k3_n5.log 2>&1
python tools/ncu_summary.py /tmp/k3_n5.ncu-rep 3638216 gpurun_out/r02b_k3_n5_ncu.txt "search node"
cp /tmp/k3_n5.ncu-rep gpurun_out/
