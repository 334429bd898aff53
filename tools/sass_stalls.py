#!/usr/bin/env python3
"""Summarise an `ncu --page source --csv --print-source sass` export: stall
samples by opcode and by reason, the hottest instructions, and memory-op
counts (LDG/LDL/STL/LDS...).  Usage: sass_stalls.py FILE[.gz] [top]"""
import csv
import gzip
import io
import sys
from collections import Counter, defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    r = csv.reader(f)
    next(r)
    hdr = next(r)
    ix = {h: k for k, h in enumerate(hdr)}
    rows = [row for row in r if len(row) == len(hdr)]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    by_op = Counter()
    by_reason = Counter()
    inst_op = Counter()
    total = 0
    hot = []
    for k, row in enumerate(rows):
        src = row[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        s = int(row[ix["Warp Stall Sampling (All Samples)"]] or 0)
        n = int(row[ix["Instructions Executed"]] or 0)
        by_op[op] += s
        inst_op[op] += n
        total += s
        for c in stall_cols:
            v = int(row[ix[c]] or 0)
            by_reason[c] += v
        hot.append((s, k, src, {c[6:]: int(row[ix[c]] or 0) for c in stall_cols if int(row[ix[c]] or 0)}))
    ninst = sum(inst_op.values())
    print(f"instructions in listing: {len(rows)}, executed (warp) {ninst}, stall samples {total}")
    print("stall reasons:")
    for c, v in by_reason.most_common(12):
        print(f"  {c:28s} {100 * v / max(total, 1):5.1f} %")
    print("by opcode (stall %, inst %):")
    for op, v in by_op.most_common(20):
        print(f"  {op:10s} {100 * v / max(total, 1):5.1f} %  {100 * inst_op[op] / max(ninst, 1):5.1f} %")
    print("memory ops executed:", {op: inst_op[op] for op in inst_op if op[:3] in ("LDG", "STG", "LDL", "STL", "LDS", "STS", "LDC", "LDGSTS")})
    print("hottest instructions:")
    for s, k, src, det in sorted(hot, reverse=True)[:top]:
        print(f"  {s:6d} #{k:5d} {src[:60]:60s} {det}")


if __name__ == "__main__":
    main()
