timeout 300 python -m pytest tests -m gpu -x -q -k "infer or predictor or dataset_votes or mnist_shaped_prefix or facade" 2>&1 | tail -2
timeout 300 python tools/infer_split.py 2>&1 | tail -14
