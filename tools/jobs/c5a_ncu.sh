ncu --set full --import-source on -k regex:mcm_batch_warp -c 1 -o gpurun_out/c5a_warp python bench.py --workload c5a --steps 1 --warmup 1 --no-cpu-baseline --no-companion --e2e-steps 0 > /dev/null 2>&1
ncu -i gpurun_out/c5a_warp.ncu-rep --page details --csv > gpurun_out/c5a_warp_details.csv 2>&1
ls -la gpurun_out/
