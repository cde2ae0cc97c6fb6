"""Build libpgmoe.so in-tree for sm_100a: ``python -m paper_2308_12066_b200.build``."""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def build(verbose: bool = False) -> str:
    csrc = os.path.join(HERE, "csrc")
    jobs = str(min(8, os.cpu_count() or 1))
    r = subprocess.run(["make", "-C", csrc, "-j", jobs], capture_output=not verbose, text=True)
    if r.returncode != 0:
        sys.stderr.write((r.stdout or "") + (r.stderr or ""))
        raise RuntimeError("libpgmoe.so build failed")
    return os.path.join(HERE, "_build", "libpgmoe.so")


if __name__ == "__main__":
    print(build(verbose=True))
