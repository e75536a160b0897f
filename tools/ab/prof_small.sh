# ncu --set full of the small per-step kernels (march count/fill, composite, adam)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^composite' -s 1 -c 1 \
  -o gpurun_out/small_full python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/small_ncu.log 2>&1; echo "ncu rc $?"
