mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for K in u 1; do
  if [ $K = u ]; then unset BSVD_VALUES_K; else export BSVD_VALUES_K=$K; fi
  echo "== K=$K"
  python bench.py --workload batch --steps 3 --warmup 3 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d.get('phases'))"
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d.get('phases'))"
done
