"""SASS opcode histogram of libnimble.so per kernel (cuobjdump -sass): evidence that the hot
paths are Blackwell-native (UTCHMMA = tcgen05.mma, UTMALDG / UTMASTG / UBLKCP = TMA, LDTM /
STTM = tcgen05.ld / st) and that no legacy HMMA (mma.sync) is used."""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2006_03031_b200/libnimble.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
keys = ("UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "LDTM", "STTM", "HMMA",
        "MUFU.EX2", "MUFU.RCP", "LDGSTS", "SYNCS.ARRIVE", "SYNCS.PHASECHK")
cur, hist = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        hist[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m:
        op = m.group(1)
        for k in keys:
            if op.startswith(k):
                hist[cur][k + (".2CTA" if ".2CTA" in op and k.startswith("UTC") else "")] += 1
print("# SASS opcode histogram of libnimble.so (cuobjdump -sass; sm_100a), per kernel instantiation")
print("# UTCHMMA(.2CTA) = tcgen05.mma, UTMALDG/UTMASTG/UBLKCP = TMA / bulk copy, LDTM/STTM = tcgen05.ld/st;")
print("# HMMA (legacy mma.sync) count is listed if present")
tot = collections.Counter()
for fn, c in hist.items():
    short = re.sub(r"^_ZN6nimble\d*", "", fn)[:110]
    print(short)
    print("    " + "  ".join(f"{k}={v}" for k, v in sorted(c.items())))
    tot.update(c)
print("TOTAL " + "  ".join(f"{k}={v}" for k, v in sorted(tot.items())))
