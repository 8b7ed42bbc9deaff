# fresh ncu captures of the final kernel 3 (n = 5 / 8 / 11) and kernel 4 (n = 5); -f: the box may keep /tmp
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=r02g
for n in 5 8 11; do
  nodes=$(python -c "import json; print(json.load(open('tests/golden/golden.json'))['dfs']['$n']['nodes'])")
  rm -f /tmp/k3_n$n.ncu-rep
  ncu -f --set full --import-source on -k regex:k3_search -s 1 -c 1 -o /tmp/k3_n$n python tools/gpu/k3_probe.py $n 2 > /tmp/k3_n$n.log 2>&1; tail -2 /tmp/k3_n$n.log
  python tools/ncu_summary.py /tmp/k3_n$n.ncu-rep $nodes gpurun_out/${TAG}_k3_n${n}_ncu.txt "search node"
done
rm -f /tmp/k4_n5.ncu-rep
ncu -f --set full --import-source on -k regex:k4_sort -s 2 -c 1 -o /tmp/k4_n5 python tools/gpu/sort_probe.py 5 > /tmp/k4_n5.log 2>&1
python tools/ncu_summary.py /tmp/k4_n5.ncu-rep 0 gpurun_out/${TAG}_k4_n5_ncu.txt
grep -h "warp instructions per\|issue_active" gpurun_out/${TAG}_k3_n*_ncu.txt
