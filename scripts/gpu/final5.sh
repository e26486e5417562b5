# round-2 final lines (after the fused copy-in): bench single / batch / reference, per-config verification
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_line.txt 2> gpurun_out/bench_err.txt
python bench.py --workload batch > gpurun_out/bench_batch_line.txt 2>> gpurun_out/bench_err.txt
python bench.py --impl reference > gpurun_out/bench_ref_line.txt 2>> gpurun_out/bench_err.txt
python scripts/verify_configs.py > gpurun_out/vc.txt 2>&1
python scripts/small_n.py > gpurun_out/small_n.txt 2>&1
tail -c 250 gpurun_out/bench_line.txt; tail -5 gpurun_out/vc.txt | cut -c1-160; cat gpurun_out/small_n.txt
