"""Run the reference's OWN test suite against the device kernels through the
INTEGRATION.md plugin stub (on the GPU box).

    python tools/run_reference_suite.py [pytest args...]

1. copies the installed, unmodified reference (baseline/_ref/tsetlinkit, pip-
   installed from /root/reference) to a scratch directory;
2. adds the stub tests/reference_backend/_b200.py as tsetlinkit/kernels/_b200.py
   and the one load_backend branch INTEGRATION.md shows -- nothing else;
3. runs the reference's tests (baseline/_ref_tests, copied from
   /root/reference/pkg/tests; git-ignored like baseline/_ref) plus
   tests/reference_backend/test_kernels_b200.py with TSETLINKIT_BACKEND=b200
   and TMB200_LIB pointing at this repo's libtmb200.so.
Writes gpurun_out/reference_suite_b200.txt (pytest output) when run there.
"""
import os
import shutil
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build(dst):
    src = os.path.join(REPO, "baseline", "_ref", "tsetlinkit")
    if not os.path.isdir(src):
        sys.exit("baseline/_ref/tsetlinkit missing: install the reference first (DESIGN.md)")
    pkg = os.path.join(dst, "tsetlinkit")
    shutil.copytree(src, pkg)
    shutil.copy(os.path.join(REPO, "tests", "reference_backend", "_b200.py"),
                os.path.join(pkg, "kernels", "_b200.py"))
    init = os.path.join(pkg, "kernels", "__init__.py")
    text = open(init).read()
    anchor = '    if name == "numba":'
    assert anchor in text, "unexpected reference kernels/__init__.py"
    text = text.replace(anchor, '    if name == "b200":\n        from . import _b200\n\n'
                                '        return _b200\n' + anchor, 1)
    open(init, "w").write(text)
    tests = os.path.join(REPO, "baseline", "_ref_tests")
    if not os.path.isdir(tests):
        sys.exit("baseline/_ref_tests missing (cp -r /root/reference/pkg/tests baseline/_ref_tests)")
    shutil.copytree(tests, os.path.join(dst, "tests"))
    shutil.copy(os.path.join(REPO, "tests", "reference_backend", "test_kernels_b200.py"),
                os.path.join(dst, "tests", "test_kernels_b200.py"))
    return dst


def main():
    dst = build(tempfile.mkdtemp(prefix="tsk_b200_"))
    env = dict(os.environ, TSETLINKIT_BACKEND="b200", PYTHONPATH=dst,
               TMB200_LIB=os.path.join(REPO, "paper_2405_04212_b200", "libtmb200.so"),
               NUMBA_CACHE_DIR=os.path.join(tempfile.gettempdir(), "numba_cache"))
    args = sys.argv[1:] or ["-q", "-p", "no:cacheprovider", "-o", "addopts="]
    cmd = [sys.executable, "-m", "pytest", os.path.join(dst, "tests")] + args
    res = subprocess.run(cmd, cwd=dst, env=env, capture_output=True, text=True)
    out = res.stdout + res.stderr
    print(out[-6000:])
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    with open(os.path.join(REPO, "gpurun_out", "reference_suite_b200.txt"), "w") as fh:
        fh.write(out)
    sys.exit(res.returncode)


if __name__ == "__main__":
    main()
