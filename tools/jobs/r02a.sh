set -x
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,memory.total --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.txt 2>&1; tail -25 $O/pytest_gpu.txt
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 600 $O/bench_c2.json
for w in c3 c4 c5a c5b; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; tail -c 300 $O/bench_$w.json; echo
done
timeout 900 python bench.py --gpus 2 --steps 3 --no-cpu-baseline > $O/bench_n2.json 2> $O/bench_n2.err; tail -c 1500 $O/bench_n2.json; tail -5 $O/bench_n2.err
