"""Recipe for oracle/_ref: the GENUINE reference package, unmodified — TEST /
BASELINE INFRASTRUCTURE ONLY.

The reference (utvkit, arXiv 2106.13402) is pure Python over numpy: there is
nothing to compile, so "building" it means copying its package directory
byte for byte from /root/reference/pkg/src/utvkit into oracle/_ref/utvkit
(git-ignored, but not gpurun-ignored, so it travels to the GPU box where
/root/reference does not exist).  A MANIFEST of sha256 digests is written
next to it and re-checked by `load()` so a modified copy is refused.

Only bench.py's reference arm (`--impl reference`, the CPU baseline) and
tests may import it; the product path never does.

    python oracle/build_ref.py        # also run by __graft_entry__.build()
"""

import hashlib
import importlib
import os
import shutil
import sys

SRC = "/root/reference/pkg/src/utvkit"
HERE = os.path.dirname(os.path.abspath(__file__))
DST_ROOT = os.path.join(HERE, "_ref")
DST = os.path.join(DST_ROOT, "utvkit")
MANIFEST = os.path.join(DST_ROOT, "MANIFEST.sha256")


def _digest(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def build():
    """Copy the reference package (no-op when /root/reference is absent)."""
    if not os.path.isdir(SRC):
        return None
    os.makedirs(DST, exist_ok=True)
    lines = []
    for name in sorted(os.listdir(SRC)):
        if not name.endswith(".py"):
            continue
        shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
        lines.append(f"{_digest(os.path.join(DST, name))}  {name}")
    with open(MANIFEST, "w") as f:
        f.write("\n".join(lines) + "\n")
    return DST


def available():
    return os.path.isfile(MANIFEST)


def load():
    """Import the copied reference as `utvkit` after checking the MANIFEST."""
    with open(MANIFEST) as f:
        for ln in f:
            dig, name = ln.split()
            if _digest(os.path.join(DST, name)) != dig:
                raise RuntimeError(f"oracle/_ref/utvkit/{name} differs from the reference copy")
    sys.dont_write_bytecode = True
    if DST_ROOT not in sys.path:
        sys.path.insert(0, DST_ROOT)
    return importlib.import_module("utvkit")


if __name__ == "__main__":
    print(build())
