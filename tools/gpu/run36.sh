timeout 900 python -m pytest tests -m gpu -x -q -k "sprm or prepass or pretrain" 2>&1 | tail -2
timeout 300 python tools/sprm_timeline.py 400000 2>&1 | grep -v Warn | tail -16
