"""Run bench.py with one tmb_set_option applied first (A/B timing):
    python tools/bench_with_option.py NAME VALUE [bench.py args...]"""
import runpy
import sys

sys.path.insert(0, ".")
from paper_2405_04212_b200 import _lib  # noqa: E402

name, value = sys.argv[1], int(sys.argv[2])
_lib.load()
_lib.call("tmb_set_option", name.encode(), value)
sys.argv = ["bench.py"] + sys.argv[3:]
runpy.run_path("bench.py", run_name="__main__")
