timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/phase_profile.py --cta 148 --epochs 4 > gpurun_out/pp.txt 2>&1
python tools/phase_profile.py --cta 148 --epochs 3 --skip 32 > gpurun_out/pp32.txt 2>&1
