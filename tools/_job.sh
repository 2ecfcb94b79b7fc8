PYTHONPATH=. timeout 900 python tools/fuzz.py 480 2>&1 | tail -8
