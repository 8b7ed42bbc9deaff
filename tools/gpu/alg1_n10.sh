# resumable exhaustive Algorithm 1 at n = 10; finished chunks -> gpurun_out/alg1_n10_new.jsonl
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B=${ALG1_BUDGET:-120}
timeout $((B + 600)) python tools/alg1_full.py 10 gpurun_out/alg1_n10_new.jsonl tests/golden/alg1_n10_chunks.jsonl --budget-s $B --chunk-leaves 2e13 2>&1 | tail -3
wc -l gpurun_out/alg1_n10_new.jsonl; tail -2 gpurun_out/alg1_n10_new.jsonl
