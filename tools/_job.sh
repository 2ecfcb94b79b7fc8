PYTHONPATH=. timeout 600 python tools/fuzz.py 420 2>&1 | tail -15
