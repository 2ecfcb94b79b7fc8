for v in lb7 lb8; do
  if [ $v != orig ]; then cp tools/libexp_$v.so paper_2008_01938_b200/_lib/libpipedp_cuda.so; fi
  timeout 600 python bench.py --workload c5b --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), d['parity']['match'])"
done
