"""Stall-sample hotspots of an ncu --set full --import-source on capture, by SASS opcode class and
by CUDA source line. Usage: ncu -i rep --page source --csv --print-source sass > src.csv;
python tools/ncu_hotspots.py src.csv  (or --page source --print-source cuda for lines)."""
import csv
import sys
from collections import Counter


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Source" in r and "Address" in r)
    i0 = rows.index(hdr)
    si, ni = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    nis = hdr.index("Warp Stall Sampling (Not-issued Samples)")
    by_op, by_op_ni, tot, tot_ni = Counter(), Counter(), 0, 0
    for r in rows[i0 + 1:]:
        if len(r) <= ni or not r[ni].strip().isdigit():
            continue
        src = r[si].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0] if not op.startswith("MUFU") else ".".join(op.split(".")[:2])
        s, sn = int(r[ni]), int(r[nis])
        by_op[op] += s
        by_op_ni[op] += sn
        tot += s
        tot_ni += sn
    print(f"stall samples: {tot} (not issued {tot_ni})")
    print(f"{'opcode':14s} {'all %':>7s} {'not-issued %':>13s}")
    for op, s in by_op.most_common(14):
        print(f"{op:14s} {100 * s / tot:7.1f} {100 * by_op_ni[op] / max(tot_ni, 1):13.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
