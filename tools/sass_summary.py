"""SASS instruction-mix summary of the built library's hot kernels
(cuobjdump -sass): the mnemonics that prove tcgen05 / TMA / dp4a / cp.async."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2410_16144_b200", "lib")
KEYS = ["UTCIMMA", "UTCQMMA", "UTCHMMA", "UTMALDG", "UBLKCP", "UTCBAR", "LDTM", "UTCATOMSWS",
        "IDP.4A", "IMMA", "HMMA", "LDGSTS", "LDGDEPBAR", "REDG", "RED", "ATOMG", "LDSM", "PRMT",
        "LOP3", "IMAD", "LDS", "STS", "LDG", "STG", "BAR", "SYNCS", "ACQBULK", "ELECT", "MEMBAR"]


def kernels(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    cur, res = None, collections.defaultdict(collections.Counter)
    for ln in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,6}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        if cur and m:
            op = m.group(1)
            res[cur]["_total"] += 1
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    res[cur][k] += 1
                    break
    return res


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return out.stdout.splitlines()


def main():
    lines = ["# SASS instruction mix (cuobjdump -sass, sm_100a build of "
             "paper_2410_16144_b200/lib)", ""]
    for obj in ("gemm_tc.o", "gemv.o", "allreduce.o"):
        res = kernels(os.path.join(LIB, obj))
        names = sorted(res)
        for n, d in zip(names, demangle(names)):
            c = res[n]
            hot = {k: v for k, v in c.items() if k != "_total" and v}
            if not hot:
                continue
            lines.append(f"## {obj}: `{d[:150]}`")
            lines.append(f"static instructions: {c['_total']}; " +
                         ", ".join(f"{k} {v}" for k, v in sorted(hot.items(), key=lambda t: -t[1])))
            lines.append("")
    text = "\n".join(lines) + "\n"
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(text)
    else:
        print(text)


if __name__ == "__main__":
    main()
