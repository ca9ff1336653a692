"""Reference CLI outputs (gen / estimate / count) for the f1/f3 parity tests.

Run in the build container: imports covcomb from /root/reference (see
make_golden.py) and writes tests/golden/cli/*.
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "cli"


def main() -> None:
    src = Path("/root/reference/pkg/src")
    dst = Path("/tmp/covcomb_golden_cli_src")
    if dst.exists():
        shutil.rmtree(dst)
    shutil.copytree(src, dst)
    sys.path.insert(0, str(dst))
    from covcomb.cli import main as ref_main

    OUT.mkdir(exist_ok=True)
    assert ref_main(["--cmd", "gen", "--n", "9", "--m", "7", "--seed", "7", "--out", str(OUT / "gen_9x7_s7.txt")]) == 0
    assert ref_main(["--cmd", "estimate", "--in", str(OUT / "gen_9x7_s7.txt"), "--p", "3", "--q", "2",
                     "--out", str(OUT / "estimate_9x7_p3q2.txt")]) == 0
    assert ref_main(["--cmd", "count", "--n", "32", "--m", "32", "--p", "13", "--q", "13",
                     "--out", str(OUT / "count_32_13.csv")]) == 0
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
