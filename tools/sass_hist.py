"""SASS instruction histograms of the hot kernels (cuobjdump -sass of the
in-tree objects; no GPU needed).  Writes profiles/<out> with, per kernel, the
total instruction count, the count per opcode (predicates and modifiers
stripped to the base mnemonic, e.g. LDS.64 kept as LDS.64), and the lines
that prove the Blackwell data path (UTMALDG / UBLKCP / SYNCS / ...).

    python tools/sass_hist.py [out_name]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1409_7166_b200", "lib")
KERNELS = [
    ("pg_sweep2.o", "_ZN3pgb11k_rb_sweep2ILi4ELi64ELb0EEEvNS_11FusedParamsE", "k_rb_sweep2<4,64> (configs 1, 3)"),
    ("pg_sweep2.o", "_ZN3pgb11k_rb_sweep2ILi8ELi32ELb0EEEvNS_11FusedParamsE", "k_rb_sweep2<8,32> (config 4)"),
    ("pg_kernels.o", "_ZN3pgb18k_csr_sweep_stagedENS_7CsrArgsE", "k_csr_sweep_staged (config 2)"),
    ("pg_kernels.o", "_ZN3pgb11k_rhs_fusedENS_7RhsArgsE", "k_rhs_fused (every config)"),
    ("pg_kernels.o", "_ZN3pgb12k_rb_clusterENS_11ClusterArgsE", "k_rb_cluster (config 0)"),
]
PROOF = ("UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "SYNCS", "FENCE", "UCGABAR", "ACQBULK", "ELECT")


def sass_of(obj, fn):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, os.path.join(LIB, obj)], capture_output=True,
                         text=True).stdout
    return out


def hist(txt):
    c = collections.Counter()
    for ln in txt.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if not m:
            continue
        t = re.sub(r"^@!?U?P\w+\s+", "", m.group(2).strip())
        op = t.split()[0]
        c[op] += 1
    return c


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "r2_sass_histograms.txt"
    lines = ["SASS instruction histograms (cuobjdump -sass of the sm_100a objects in "
             "paper_1409_7166_b200/lib; static counts over the whole function body)", ""]
    for obj, fn, label in KERNELS:
        txt = sass_of(obj, fn)
        c = hist(txt)
        if not c:
            lines.append(f"== {label}: not found ({fn})")
            continue
        tot = sum(c.values())
        lines.append(f"== {label}  [{fn}]  total {tot} instructions")
        fam = collections.Counter()
        for op, v in c.items():
            fam[op.split(".")[0]] += v
        lines.append("  by family: " + ", ".join(f"{k} {v}" for k, v in fam.most_common(24)))
        lines.append("  by opcode: " + ", ".join(f"{k} {v}" for k, v in c.most_common(40)))
        proof = {k: v for k, v in c.items() if k.split(".")[0] in PROOF}
        lines.append("  Blackwell data path: " + (", ".join(f"{k} {v}" for k, v in sorted(proof.items()))
                                                  or "none"))
        lines.append("")
    out = os.path.join(ROOT, "profiles", name)
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
