python -m pytest tests/test_gpu_sdp.py -m gpu -x -q -k "progressive or config2 or chunked" 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 > gpurun_out/prog_bench.json 2> gpurun_out/prog_bench.err; tail -c 1500 gpurun_out/prog_bench.json
