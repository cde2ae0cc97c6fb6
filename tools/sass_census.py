"""SASS instruction census of every kernel in libpgmoe.so: counts of the
mnemonics that evidence tcgen05 (UTC*MMA, LDTM), TMA (UTMALDG / UBLKCP),
FP64 routing (DFMA) and the synchronisation used.
    python tools/sass_census.py [lib.so] > profiles/r2/sass_census.txt"""
import collections
import re
import subprocess
import sys

KEEP = re.compile(r"^(UTC\w*MMA|UTCBAR|LDTM|STTM|UTMALDG|UTMASTG|UTMAPF|UBLKCP|DFMA|DADD|DMUL|F2F|SYNCS|ELECT|"
                  r"MATCH|MEMBAR|FENCE|ATOMG|ATOM|RED|LDG|STG|LDS|STS|HMMA|BAR|NANOSLEEP)")


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else "paper_2308_12066_b200/_build/libpgmoe.so"
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    fn, counts, out = None, collections.Counter(), []
    for ln in sass.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            if fn:
                out.append((fn, counts))
            fn, counts = m.group(1), collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        if m and fn:
            op = m.group(1)
            base = op.split(".")[0]
            if KEEP.match(base):
                counts[op if base in ("UTMALDG", "UBLKCP") else base] += 1
    if fn:
        out.append((fn, counts))
    names = subprocess.run(["c++filt"], input="\n".join(f for f, _ in out), capture_output=True, text=True).stdout.split("\n")
    print(f"# SASS census of {so} (cuobjdump -sass), sm_100a")
    for (f, c), dn in zip(out, names):
        print(f"{dn[:150]}\n   " + " ".join(f"{k}={v}" for k, v in sorted(c.items())))


if __name__ == "__main__":
    main()
