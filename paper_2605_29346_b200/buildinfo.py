"""Build provenance of libgnnb200.so.

The source hash is sha256 over every file that goes into the library
(``csrc/*.cu``, ``csrc/*.cuh``, ``csrc/Makefile``, ``include/*.h``) in sorted
order.  ``make`` embeds it (``gnn_build_id()``), and ``smoke()`` / bench.py
recompute it from the files that travelled with the snapshot: a library that
was not built from exactly these sources is refused, so a stale prebuilt
``.so`` cannot pass for the current code.  No torch import here: the Makefile
runs this file as a script.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)


def source_files() -> list[str]:
    csrc = os.path.join(PKG, "csrc")
    inc = os.path.join(ROOT, "include")
    out = [os.path.join(csrc, f) for f in os.listdir(csrc)
           if f.endswith((".cu", ".cuh")) or f == "Makefile"]
    out += [os.path.join(inc, f) for f in os.listdir(inc) if f.endswith(".h")]
    return sorted(out, key=lambda p: os.path.relpath(p, ROOT))


def source_hash() -> str:
    h = hashlib.sha256()
    for p in source_files():
        h.update(os.path.relpath(p, ROOT).encode() + b"\0")
        with open(p, "rb") as f:
            h.update(f.read())
        h.update(b"\0")
    return h.hexdigest()[:16]


def git_sha() -> str:
    try:
        out = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"],
                             capture_output=True, text=True, timeout=10)
        dirty = subprocess.run(["git", "-C", ROOT, "status", "--porcelain", "--",
                                "paper_2605_29346_b200/csrc", "include"],
                               capture_output=True, text=True, timeout=10)
        sha = out.stdout.strip() if out.returncode == 0 else "nogit"
        return sha + ("+dirty" if dirty.stdout.strip() else "")
    except Exception:
        return "nogit"


def write_header(path: str) -> None:
    """build/build_id.h, rewritten only when the id changes (so make only
    recompiles abi.cu when a source changed)."""
    text = (f'#define GNN_SRC_HASH "{source_hash()}"\n'
            f'#define GNN_GIT_SHA "{git_sha()}"\n')
    try:
        with open(path) as f:
            if f.read() == text:
                return
    except OSError:
        pass
    with open(path, "w") as f:
        f.write(text)


if __name__ == "__main__":
    if len(sys.argv) == 3 and sys.argv[1] == "--header":
        write_header(sys.argv[2])
    else:
        print(source_hash())
