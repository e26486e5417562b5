# round-end evidence: bench lines, per-config verification, launch list, ncu summaries, traffic
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_line.txt 2> gpurun_out/bench_err.txt
python bench.py --impl reference > gpurun_out/bench_ref_line.txt 2>> gpurun_out/bench_err.txt
python bench.py --workload batch > gpurun_out/bench_batch_line.txt 2>> gpurun_out/bench_err.txt
python scripts/verify_configs.py > gpurun_out/vc.txt 2>&1
python scripts/traffic_capture.py 8192 > gpurun_out/traffic.txt 2>&1
bash scripts/gpu/prof_r02b.sh > gpurun_out/prof_b.log 2>&1
tail -c 1500 gpurun_out/bench_line.txt; tail -c 600 gpurun_out/bench_ref_line.txt; tail -c 600 gpurun_out/bench_batch_line.txt
