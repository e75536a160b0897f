# Round-end measurement, part B: one ncu --set full capture of the four field kernels
# (after the same command exits 0 without ncu).
python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/final_b1.json 2>&1; echo "b1 rc $?"
ncu --set full --clock-control none --import-source on -k regex:'field_(gather|fwd|bwd|scatter)' -c 4 -o gpurun_out/final_full python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/final_full.log 2>&1; echo "ncu rc $?"
