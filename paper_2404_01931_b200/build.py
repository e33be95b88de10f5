"""Builds libflipb200.so in-tree (nvcc, sm_100a only)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")


def build(jobs: int = 8) -> str:
    subprocess.run(["make", "-s", "-C", CSRC, f"-j{jobs}"], check=True)
    return os.path.join(HERE, "libflipb200.so")


if __name__ == "__main__":
    print(build())
