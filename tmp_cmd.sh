timeout 600 python -m pytest tests -m gpu -x -q -k "mnist or keyed or train_small or multi_cta or block_layouts" 2>&1 | tail -2
python tools/phase_profile.py --cta 148 --epochs 4 > gpurun_out/pp.txt 2>&1
