O=gpurun_out/r02h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sdp.py -m gpu -q -x > $O/pytest_sdp.txt 2>&1; tail -3 $O/pytest_sdp.txt
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -m gpu -q > $O/pytest_sanitizer.txt 2>&1; tail -5 $O/pytest_sanitizer.txt
cp gpurun_out/sanitizer_*.txt $O/ 2>/dev/null
for f in $O/sanitizer_*; do echo $f; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ALL OK" $f; done
