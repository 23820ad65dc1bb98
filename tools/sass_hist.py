"""SASS opcode histogram of the library's kernels (cuobjdump -sass), written as JSON: per
kernel the opcode counts plus the Blackwell-native evidence (UTC*MMA = tcgen05.mma,
UTMALDG/UTMASTG = TMA, LDTM/STTM = tcgen05.ld/st, POPC, multimem stores).
Usage: python tools/sass_hist.py <.so|.o|.cubin> [name-filter] > profiles/<round>_sass_hist.json"""
import collections
import json
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
pat = sys.argv[2] if len(sys.argv) > 2 else ""
fn = None
hist = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        fn = m.group(1)
        hist[fn] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and fn:
        hist[fn][m.group(1).split(".")[0]] += 1
KEYS = ("UTCQMMA", "UTCOMMA", "UTCIMMA", "UTCHMMA", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "LDTM", "STTM",
        "POPC", "LOP3", "IMMA", "HMMA")
res = {"binary": sys.argv[1], "kernels": {}}
tot = collections.Counter()
for f, h in hist.items():
    if pat not in f or not sum(h.values()):
        continue
    res["kernels"][f] = {"instructions": sum(h.values()), "evidence": {k: h[k] for k in KEYS if h[k]},
                         "top": dict(h.most_common(12))}
    tot.update(h)
res["total_evidence"] = {k: tot[k] for k in KEYS if tot[k]}
print(json.dumps(res, indent=1))
