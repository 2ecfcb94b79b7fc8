PYTHONPATH=. timeout 900 python tools/fuzz.py 600 2>&1 | tail -8
