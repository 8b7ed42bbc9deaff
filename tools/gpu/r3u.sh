# final GPU suite + smoke on the session's last commit
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3u_smoke.log 2>&1; tail -1 gpurun_out/r3u_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r3u_gpu_tests.log 2>&1; tail -3 gpurun_out/r3u_gpu_tests.log
