# A/B: exact-n flattened (facet, ridge) passes vs the power-of-two lanes per
# facet; single-GPU pre-split depth at n = 5; n = 5 source-level ncu breakdown
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_REPS=9 timeout 900 python tools/ab_k3.py 5,6,8,11 ":" "exn:" ":" "exn:" > gpurun_out/r3b_ab_exn.jsonl 2>&1; cat gpurun_out/r3b_ab_exn.jsonl
timeout 300 python tools/gpu/split_n5.py 5 > gpurun_out/r3b_split_n5.txt 2>&1; cat gpurun_out/r3b_split_n5.txt
ncu --set full --import-source on -k regex:k3_search -s 1 -c 1 -o /tmp/k3_n5 python tools/gpu/k3_probe.py 5 2 > /tmp/k3_n5.log 2>&1
python tools/ncu_breakdown.py /tmp/k3_n5.ncu-rep 3638216 > gpurun_out/r3b_k3_n5_breakdown.txt 2>&1; head -40 gpurun_out/r3b_k3_n5_breakdown.txt
ncu -i /tmp/k3_n5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r3b_k3_n5_source.csv 2>/dev/null; ls -la gpurun_out/r3b_k3_n5_source.csv
timeout 120 python tools/e2e_trace.py 5 > gpurun_out/r3b_e2e_trace.txt 2>&1; tail -40 gpurun_out/r3b_e2e_trace.txt
