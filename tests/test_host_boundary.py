"""The product boundary (CPU-only checks): no CPU fallback and no oracle on
the product path.

* importing the package without its CUDA library fails loudly (ImportError
  naming the build command) instead of degrading to a host path;
* nothing under paper_2402_12274_b200/ (Python or C++/CUDA sources) imports,
  links or loads oracle/ -- the oracle is test infrastructure only."""

import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2402_12274_b200")


def test_import_without_libmpx_fails_loudly(tmp_path):
    env = dict(os.environ, MPX_LIB_PATH=str(tmp_path / "missing" / "libmpx.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_2402_12274_b200"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "ImportError" in r.stderr and "no CPU fallback" in r.stderr


def test_product_never_references_the_oracle():
    pat = re.compile(r"\boracle\b|dt_oracle|brute\.py")
    offenders = []
    for d, _, files in os.walk(PKG):
        if "_obj" in d or "__pycache__" in d:
            continue
        for f in files:
            if not f.endswith((".py", ".cu", ".cpp", ".hpp", ".cuh", ".h")):
                continue
            p = os.path.join(d, f)
            with open(p, encoding="utf-8", errors="replace") as fh:
                for i, line in enumerate(fh, 1):
                    code = line.split("#")[0] if f.endswith(".py") else line.split("//")[0]
                    if pat.search(code):
                        offenders.append("%s:%d: %s" % (os.path.relpath(p, ROOT), i, line.strip()))
    assert not offenders, offenders
