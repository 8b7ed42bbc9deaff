# n = 11 TS class: 24 warps x 64 frames (base) vs 27 / 26 warps x 40 frames; drop-in conversion on the host pool
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_REPS=9 timeout 900 python tools/ab_k3.py 11 ":" "c11:" "c11b:" ":" "c11:" "c11b:" > gpurun_out/r3g_ab_c11.jsonl 2>&1; cat gpurun_out/r3g_ab_c11.jsonl
./build/dropin_e2e 5 0 9 > gpurun_out/r3g_dropin5.json 2>&1; cat gpurun_out/r3g_dropin5.json
./build/dropin_e2e 8 0 5 > gpurun_out/r3g_dropin8.json 2>&1; cat gpurun_out/r3g_dropin8.json
