timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 1500 python -m paper_2508_06339_b200 accuracy --sizes 1024,4096 --precisions fp64,fp32,fp16 --per-distribution 2 --output gpurun_out/accuracy_1024_4096.csv > gpurun_out/acc1.log 2>&1; cat gpurun_out/accuracy_1024_4096.csv
timeout 1500 python -m paper_2508_06339_b200 accuracy --sizes 16384 --precisions fp64,fp32,fp16 --per-distribution 1 --output gpurun_out/accuracy_16384.csv > gpurun_out/acc2.log 2>&1; cat gpurun_out/accuracy_16384.csv; tail -3 gpurun_out/acc2.log
timeout 1500 python -m paper_2508_06339_b200 tune --sizes 4096,8192 --tilesizes 32,64,128 --precision fp32 --batch 3 --min-total 0 --output gpurun_out/tune_fp32.csv > gpurun_out/tune.log 2>&1; cat gpurun_out/tune_fp32.csv; tail -3 gpurun_out/tune.log
