# re-entry check: the full GPU suite twice, smoke(), one bench line
for k in 1 2; do
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_all_$k.log 2>&1; echo "all gpu run $k rc $?"; grep -E "^FAILED|passed|failed" gpurun_out/gpu_all_$k.log | tail -8
done
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_re.json 2> gpurun_out/bench_re.err; tail -c 600 gpurun_out/bench_re.json
