"""The product path has no fallback: it never reaches oracle/ and fails loudly without libmgnn.so.

Host-only checks (-m "not gpu"): a static scan of the package sources, and the binding's loader
run in a fresh interpreter with the library path pointed at a file that does not exist.
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2410_22697_b200")


def _package_sources():
    for d, _, files in os.walk(PKG):
        if "build" in d.split(os.sep) or "__pycache__" in d:
            continue
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                yield os.path.join(d, f)


def test_package_never_references_oracle():
    pat = re.compile(r"\boracle\b|liborc")
    hits = []
    for p in _package_sources():
        with open(p, encoding="utf-8") as fh:
            for i, line in enumerate(fh, 1):
                code = line.split("#", 1)[0] if p.endswith(".py") else line.split("//", 1)[0]
                if pat.search(code):
                    hits.append(f"{os.path.relpath(p, ROOT)}:{i}: {line.strip()}")
    assert not hits, "product sources reference the oracle:\n" + "\n".join(hits)


def test_missing_library_raises():
    code = ("import paper_2410_22697_b200._lib as L\n"
            "try:\n    L.load()\nexcept ImportError as e:\n    print('RAISED', e)\n"
            "else:\n    print('LOADED')\n")
    env = dict(os.environ, MGNN_LIB=os.path.join(ROOT, "no_such_dir", "libmgnn.so"))
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("RAISED"), out.stdout
