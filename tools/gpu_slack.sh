# A/B: predicted-exponent slack 10 (default) vs 0, c2 field-backward diagnostic
python tools/diag_c2.py > gpurun_out/diag_slack10.log 2>&1
NS2B_NVCC_EXTRA=-DNS2B_PRED_SLACK=0 python -m paper_2212_05231_b200.build --force > /dev/null
python tools/diag_c2.py > gpurun_out/diag_slack0.log 2>&1
grep -A1 "^dc_only\|^full" gpurun_out/diag_slack10.log gpurun_out/diag_slack0.log
