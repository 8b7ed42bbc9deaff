# (1) 32-bit node counter + 32-bit open-ridge prune (main) vs the previous commit (prev);
# (2) map-queue classes at n = 9, 10: 16 warps x 2 CTAs (prev) vs 20 x 2 (48 regs) vs 18 x 2 with 40 frames
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_REPS=7 timeout 1200 python tools/ab_k3.py 5,8,11 "prev:" ":" "prev:" ":" > gpurun_out/r3h_ab_cnt.jsonl 2>&1; cat gpurun_out/r3h_ab_cnt.jsonl
AB_REPS=7 timeout 1200 python tools/ab_k3.py 9,10 "prev:" "mq20:" "mq18:" "prev:" "mq20:" "mq18:" > gpurun_out/r3h_ab_mq.jsonl 2>&1; cat gpurun_out/r3h_ab_mq.jsonl
