for sd in 0 60 120 126; do BSVD_FPANEL_TRACE=gpurun_out/tr_$sd.txt BSVD_FPANEL_TRACE_SIDE=$sd python scripts/prof_one.py 8192; done
cat gpurun_out/tr_*.txt
