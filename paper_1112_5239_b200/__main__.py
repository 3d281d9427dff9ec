"""Command-line emitter: stream generated words to standard output (or a
file) for external test batteries -- SPEC S:378 "raw little-endian 32-bit
words to file or standard output"; the paper ran TestU01 BigCrush on its
generators.

    python -m paper_1112_5239_b200 --variant 1 --streams 1048576 --n 128 \\
        --calls 8 [--format raw-le32|hex|bits] [--seed S] [--out FILE] | consumer

Each call is one prng_emit: n rounds of every stream, stream-major.
"""
from __future__ import annotations

import argparse
import sys

import torch

from . import EMIT_FORMATS, ChaoticPRNG


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1112_5239_b200", description=__doc__.split("\n\n")[0])
    ap.add_argument("--variant", type=int, default=1, choices=range(5))
    ap.add_argument("--seed", type=lambda v: int(v, 0), default=0x0123456789ABCDEF)
    ap.add_argument("--streams", type=int, default=1 << 20)
    ap.add_argument("--n", type=int, default=128, help="rounds per stream per call")
    ap.add_argument("--calls", type=int, default=1)
    ap.add_argument("--format", choices=sorted(EMIT_FORMATS), default="raw-le32")
    ap.add_argument("--out", default=None, help="file (default: standard output)")
    ap.add_argument("--paper-defaults", action="store_true", help="V0, one stream: Listing 1's initial state")
    a = ap.parse_args(argv)
    torch.cuda.set_device(0)
    g = ChaoticPRNG(a.seed, a.streams, a.variant, paper_defaults=a.paper_defaults)
    total = 0
    if a.out is None:
        sys.stdout.flush()
        fd = sys.stdout.fileno()
        for _ in range(a.calls):
            total += g.emit(a.n, fd, a.format)
    else:
        with open(a.out, "wb") as fh:
            for _ in range(a.calls):
                total += g.emit(a.n, fh, a.format)
    g.close()
    print(f"emitted {total} bytes", file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())
