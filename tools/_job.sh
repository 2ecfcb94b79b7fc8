timeout 600 python -m pytest tests/test_gpu_sdp.py -x -q -k "chunked" 2>&1 | tail -2
timeout 300 python bench.py --workload c2 --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), (d['parity'] or {}).get('match'), d['roofline']['kernel'], d['gpu_launches'], d['relaxation_roofline']['frac'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launch_chunked.csv python bench.py --workload c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python - <<'P'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launch_chunked.csv")))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if len(r) > 5 and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        nm = r[hdr.index("Kernel Name")].split("(")[0][:60]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        a = agg.setdefault(nm, [0, 0.0]); a[0] += 1; a[1] += v
for k, (c, t) in agg.items(): print(f"{k:60s} {c:5d} {t/1e6:9.3f} ms")
P
