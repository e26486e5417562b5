# new chase-protocol tests + per-config verification (warm) 
python -m pytest tests/test_gpu_configs.py -x -q -k "mailbox or wide_tile" 2>&1 | tail -2
python scripts/verify_configs.py > gpurun_out/vc.txt 2>&1; tail -5 gpurun_out/vc.txt
