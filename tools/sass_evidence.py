"""Per-kernel SASS mnemonic counts of the built library (cuobjdump -sass):
the evidence that the hot kernels use what DESIGN.md says they use -- TMA
bulk tensor stores (UTMASTG), swizzled STS.128 staging, warp shuffles for
the neighbour exchange (SHFL.IDX), shared-memory histogram atomics (ATOMS),
and the integer pipes (LOP3 / SHF on ALU, IMAD / IMAD.HI / IMAD.WIDE on FMA).

  python tools/sass_evidence.py > profiles/<tag>_sass_evidence.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1112_5239_b200", "libciprng.so")
KEYS = ["UTMASTG", "UBLKCP", "STS.128", "STG.E.128", "STG.E", "LDG", "LDS", "SHFL.IDX", "ATOMS", "RED", "PRMT", "LOP3", "SHF",
        "IMAD.HI", "IMAD.WIDE", "IMAD.SHL", "IMAD", "VIADDMNMX", "VIMNMX", "FFMA", "DFMA", "BMSK"]
# kernels behind the bench rows (demangled-name prefixes, store/consume instantiations)
SHOW = ["v1_fast_kernel<ciprng::StoreSink, 32, 2, false>", "v1_band_kernel<2, 2>",
        "v1_fast_kernel<ciprng::StatsSink", "v1_fast_kernel<ciprng::StatsSinkCtaT<2>", "v1_fast_kernel<ciprng::BatterySinkT<true>",
        "comb_fast_kernel<ciprng::SrcXor64T<0>, ciprng::StatsSinkCtaT<2>", "comb_fast_kernel<ciprng::SrcXor64T<0>, ciprng::StoreSink, 32, false>",
        "comb_fast_kernel<ciprng::SrcXor64T<0>, ciprng::StatsSink", "v0_kernel<ciprng::StoreSink, false, 0>",
        "v0_kernel<ciprng::StoreSink, true, 0>", "v2_kernel<ciprng::StoreSink, 0u, true>",
        "v2_kernel<ciprng::StoreSink, 256u, true>", "v2_kernel<ciprng::StatsSink", "cbg_encrypt_kernel",
        "alg1_kernel", "v0_jump_kernel", "digest_kernel", "format_kernel"]


def main():
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs, cur = collections.OrderedDict(), None
    for ln in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            cur = funcs.setdefault(name, collections.Counter())
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        if m and cur is not None:
            op = m.group(1)
            for k in KEYS:  # first (most specific) matching key
                if op == k or op.startswith(k + "."):
                    cur[k] += 1
                    break
    print("# SASS evidence (cuobjdump -sass paper_1112_5239_b200/libciprng.so, sm_100a)\n")
    print("Static instruction counts per kernel (whole function, not per number).\n")
    print("| kernel | " + " | ".join(KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for want in SHOW:
        for name, c in funcs.items():
            short = name.replace("void ", "").split("(")[0].replace("ciprng::", "")
            if want.replace("ciprng::", "") in short:
                print(f"| `{short}` | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + " |")
                break


if __name__ == "__main__":
    sys.exit(main())
