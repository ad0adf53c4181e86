"""Build ``oracle/_ref``: the reference package compiled to bytecode.

TEST INFRASTRUCTURE ONLY (never imported by the product path).

The reference (``/root/reference/pkg/src/bdem``) is pure Python, so its
"build" is byte compilation: every module is compiled from the sources where
they lie into a sourceless ``.pyc`` and the package is stored as the zip
archive ``oracle/_ref/bdem_ref.zip`` (git-ignored, not gpurun-ignored -- it
travels to the GPU box like ``lib/*.so``; loose ``.pyc`` files do not).  No
source text is copied.  On the GPU box, where ``/root/reference`` does not
exist, the tests and ``bench.py --impl reference`` import the UNMODIFIED
reference from there through ``zipimport``:

    sys.path.insert(0, "oracle/_ref/bdem_ref.zip"); import bdem

The bytecode is tied to the interpreter version (3.12 here and on the box:
same image); ``load()`` checks the magic number and returns None on a
mismatch so callers can skip with a reason.
"""

from __future__ import annotations

import importlib.util
import os
import py_compile
import sys
import tempfile
import zipfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src/bdem"
OUT = os.path.join(HERE, "_ref")
ZIP = os.path.join(OUT, "bdem_ref.zip")
STAMP = os.path.join(OUT, "MAGIC")


def build(src: str = REF_SRC) -> str | None:
    """Compile every reference module and archive the package as
    ``oracle/_ref/bdem_ref.zip`` (``bdem/<name>.pyc`` entries).

    Returns the archive path, or None when the reference sources are absent
    (the GPU box: it uses the prebuilt archive)."""
    if not os.path.isdir(src):
        return None
    os.makedirs(OUT, exist_ok=True)
    names = sorted(f for f in os.listdir(src) if f.endswith(".py"))
    with tempfile.TemporaryDirectory() as tmp:
        tmp_zip = os.path.join(tmp, "bdem_ref.zip")
        with zipfile.ZipFile(tmp_zip, "w", zipfile.ZIP_DEFLATED) as zf:
            for f in names:
                pyc = os.path.join(tmp, f[:-3] + ".pyc")
                py_compile.compile(os.path.join(src, f), cfile=pyc, doraise=True,
                                   invalidation_mode=py_compile.PycInvalidationMode.UNCHECKED_HASH)
                zf.write(pyc, "bdem/" + f[:-3] + ".pyc")
        os.replace(tmp_zip, ZIP)
    with open(STAMP, "w") as fh:
        fh.write(importlib.util.MAGIC_NUMBER.hex() + "\n")
    return ZIP


def available() -> bool:
    try:
        with open(STAMP) as fh:
            return fh.read().strip() == importlib.util.MAGIC_NUMBER.hex()
    except OSError:
        return False


def load():
    """Import the reference ``bdem`` package: the bytecode build if present
    (the GPU box), else the sources (this container); None if neither."""
    if "bdem" in sys.modules:
        return sys.modules["bdem"]
    if available() and os.path.exists(ZIP):
        sys.path.insert(0, ZIP)
    elif os.path.isdir(REF_SRC):
        sys.dont_write_bytecode = True
        sys.path.insert(0, os.path.dirname(REF_SRC))
    else:
        return None
    import bdem
    import bdem.solver  # noqa: F401
    return bdem


if __name__ == "__main__":
    print(build())
