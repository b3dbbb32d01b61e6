"""Install the UNMODIFIED reference (tsetlinkit) into the git-ignored
baseline/_ref and copy its own tests to baseline/_ref_tests, as DESIGN.md §6
records.  /root/reference is read-only, so the wheel is built from a copy
under /tmp.  Called by __graft_entry__.build() when /root/reference is
present and the install is missing (baseline/_ref travels to the GPU box;
/root/reference does not)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg"


def install(force: bool = False) -> bool:
    dst = os.path.join(REPO, "baseline", "_ref")
    tests = os.path.join(REPO, "baseline", "_ref_tests")
    if not os.path.isdir(SRC):
        return False
    if force or not os.path.isdir(os.path.join(dst, "tsetlinkit")):
        shutil.rmtree(dst, ignore_errors=True)
        os.makedirs(dst, exist_ok=True)
        with tempfile.TemporaryDirectory(prefix="tsetlinkit_src_") as tmp:
            work = os.path.join(tmp, "pkg")
            shutil.copytree(SRC, work)
            subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index",
                            "--no-build-isolation", "--no-deps", "--find-links",
                            "/opt/wheelhouse", "--target", dst, work], check=True)
    if force or not os.path.isdir(tests):
        shutil.rmtree(tests, ignore_errors=True)
        shutil.copytree(os.path.join(SRC, "tests"), tests)
    return True


if __name__ == "__main__":
    print("installed" if install(force="--force" in sys.argv) else "no /root/reference here")
