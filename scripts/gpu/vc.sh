mkdir -p gpurun_out
for p in 2 4 8; do BSVD_SLICE_PER=$p TAG=slice$p python scripts/s3_time.py 8192 u; done
BSVD_SLICE_PER=2 TAG=slice2 python scripts/s3_time.py 16384 u
TAG=slice4 python scripts/s3_time.py 16384 u
python scripts/verify_configs.py > gpurun_out/vc.txt 2>&1
python scripts/verify_configs.py c1 c2 >> gpurun_out/vc.txt 2>&1
cat gpurun_out/vc.txt | cut -c1-400
