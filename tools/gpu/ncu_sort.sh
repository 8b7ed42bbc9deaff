cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for n in 5 8; do
WPM_BUCKET_TILE=1024 ncu --set full --import-source on -k regex:k4_bucket -s 2 -c 1 -o /tmp/kb_n$n python tools/gpu/sort_probe.py $n > /tmp/kb_n$n.log 2>&1
python tools/ncu_summary.py /tmp/kb_n$n.ncu-rep 0 gpurun_out/kb_n${n}_ncu.txt
WPM_SORT=merge ncu --set full --import-source on -k regex:k4_sort -s 2 -c 1 -o /tmp/km_n$n python tools/gpu/sort_probe.py $n > /tmp/km_n$n.log 2>&1
python tools/ncu_summary.py /tmp/km_n$n.ncu-rep 0 gpurun_out/km_n${n}_ncu.txt
done
ncu -i /tmp/kb_n5.ncu-rep --page source --csv --print-source cuda > gpurun_out/kb_n5_src.csv 2>&1
ncu -i /tmp/kb_n8.ncu-rep --page source --csv --print-source cuda > gpurun_out/kb_n8_src.csv 2>&1
