mkdir -p gpurun_out/ncu
run() { name=$1; units=$2; uname=$3; shift 3; ncu --set full --import-source on -o /tmp/$name "$@" > /tmp/$name.log 2>&1; tail -1 /tmp/$name.log; python tools/ncu_summary.py /tmp/$name.ncu-rep $units gpurun_out/ncu/$name.txt "$uname"; }
run k1_n11 0 launch -k regex:k1_universe -s 1 -c 1 python tools/gpu/kernels_probe.py create 11
run k2_n11 0 launch -k regex:k2_incidence -s 1 -c 1 python tools/gpu/kernels_probe.py create 11
run k2_n5 0 launch -k regex:k2_incidence -s 1 -c 1 python tools/gpu/kernels_probe.py create 5
run k3_n5 3638216 "search node" -k regex:k3_search -s 1 -c 1 python tools/gpu/kernels_probe.py k3 5
run k3_n8 126316850 "search node" -k regex:k3_search -s 1 -c 1 python tools/gpu/kernels_probe.py k3 8
run k3_n11 38438253 "search node" -k regex:k3_search -s 1 -c 1 python tools/gpu/kernels_probe.py k3 11
run k4_n5 242043 row -k regex:k4_sort -s 1 -c 1 python tools/gpu/kernels_probe.py k3 5
run k4_n8 1719929 row -k regex:k4_sort -s 1 -c 1 python tools/gpu/kernels_probe.py k3 8
run k5_remap_n5 242043 row -k regex:remap_rows -s 1 -c 1 python tools/gpu/kernels_probe.py line13 5
run k5_filter_n5 202984 row -k regex:filter_rows -s 1 -c 1 python tools/gpu/kernels_probe.py line13 5
run k6_n7 17304607848 leaf -k regex:odometer -s 1 -c 1 python tools/gpu/kernels_probe.py alg1 7
run k8_n11 154527 row -k regex:k8_verify -s 1 -c 1 python tools/gpu/kernels_probe.py verify 11
cp /tmp/k3_n5.ncu-rep /tmp/k4_n8.ncu-rep gpurun_out/ncu/
python bench.py --steps 2 --warmup 3 --no-per-n --no-cpu-baseline > gpurun_out/ncu/bench_plain.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches.csv python bench.py --steps 2 --warmup 3 --no-per-n --no-cpu-baseline > gpurun_out/ncu/launch.log 2>&1
python tools/ncu_summary.py --launches gpurun_out/ncu/launches.csv 2 gpurun_out/ncu/launches.txt
du -sh gpurun_out
