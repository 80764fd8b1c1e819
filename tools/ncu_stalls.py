"""Summarise warp-stall sampling of one kernel from an ncu report's SASS source page:
    ncu -i prof.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_stalls.py src.csv "title" > profiles/rNN_<kernel>_stalls.md
Totals by stall reason and by opcode, and the top instructions with their main reason."""
import csv
import sys
from collections import defaultdict


def main(path, title):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    si = hdr.index("Source")
    ti = hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [(i, h[len("stall_"):]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    by_reason, by_op, insts = defaultdict(int), defaultdict(int), []

    def num(x):
        try:
            return int(float(x.replace(",", "")))
        except ValueError:
            return 0

    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr):
            continue
        tot = num(r[ti])
        if not tot:
            continue
        per = {name: num(r[i]) for i, name in reasons}
        for k, v in per.items():
            by_reason[k] += v
        src = r[si].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        by_op[op.split(".")[0]] += tot
        insts.append((tot, src, max(per, key=per.get)))
    total = sum(by_reason.values())
    print(f"# {title}\n\nTotal samples: {total}\n\n## By stall reason\n\n| reason | samples |\n|---|---|")
    for k, v in sorted(by_reason.items(), key=lambda kv: -kv[1])[:10]:
        print(f"| {k} | {v} |")
    print("\n## By opcode\n\n| opcode | samples |\n|---|---|")
    for k, v in sorted(by_op.items(), key=lambda kv: -kv[1])[:12]:
        print(f"| {k} | {v} |")
    print("\n## Top instructions\n\n| samples | instruction | main reason |\n|---|---|---|")
    for tot, src, why in sorted(insts, reverse=True)[:20]:
        print(f"| {tot} | `{src}` | {why} |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "warp-stall sampling")
