# flakiness check: the full GPU suite twice, then smoke()
for k in 1 2; do
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_all_$k.log 2>&1; echo "all gpu run $k rc $?"; grep -E "^FAILED|passed|failed" gpurun_out/gpu_all_$k.log | tail -8
done
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
