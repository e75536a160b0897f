NS2B_NVCC_EXTRA=-DNS2B_PHASE_PROF python -m paper_2212_05231_b200.build --force > /dev/null
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu 2>/dev/null | grep PHASEPROF | tail -3
python -m paper_2212_05231_b200.build --force > /dev/null
