"""Build the oracle's C restatement (oracle/_lib/libforest_oracle.so).

Test infrastructure only: used by bench.py's CPU-baseline legs and tests.
"""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_lib", "libforest_oracle.so")


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "forest_oracle.c")
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= os.path.getmtime(src):
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC", "-o", OUT,
                    src], check=True)
    return OUT


if __name__ == "__main__":
    print(build(force=True))
