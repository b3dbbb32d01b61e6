timeout 600 python -m pytest tests -m gpu -x -q -k "sparse" 2>&1 | tail -2
timeout 600 python tools/sparse_phase.py 2>&1 | tail -7
