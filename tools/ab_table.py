#!/usr/bin/env python
"""Table of a tools/cm_mid2.py-style A/B jsonl: flushed / back-to-back µs per
shape (rows) and tag (columns), mean over repeated runs of the same tag."""
import json
import sys
from collections import defaultdict

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
tags, shapes, acc = [], [], defaultdict(list)
for r in rows:
    k = (r["dtype"].replace("float", "f"), r["m"], r["n"])
    if r["tag"] not in tags:
        tags.append(r["tag"])
    if k not in shapes:
        shapes.append(k)
    acc[(r["tag"], k)].append((r["flushed_us"], r["b2b_us"]))
print("shape".ljust(22), " ".join(t.rjust(13) for t in tags))
for k in shapes:
    line = str(k).ljust(22)
    for t in tags:
        v = acc.get((t, k))
        line += " " + (f"{sum(a for a, _ in v) / len(v):.1f}/{sum(b for _, b in v) / len(v):.1f}" if v else "-").rjust(13)
    print(line)
