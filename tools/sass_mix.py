"""Instruction mix and stall samples per SASS opcode from an ncu
`--page source --csv` export (one kernel):

    python tools/sass_mix.py gpurun_out/X_source.csv [top]
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hdr = rows[1]
    i_src, i_stall, i_ex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
        hdr.index("Instructions Executed")
    ex = collections.Counter()
    st = collections.Counter()
    for r in rows[2:]:
        if len(r) <= i_ex or not r[i_ex].strip():
            continue
        op = r[i_src].split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1] if len(op) > 1 else o
        o = o.split(".")[0]
        ex[o] += int(r[i_ex].replace(",", "") or 0)
        st[o] += int(r[i_stall].replace(",", "") or 0)
    te, ts = sum(ex.values()), sum(st.values())
    print(f"total warp instructions {te:,}  stall samples {ts:,}")
    for o, n in ex.most_common(top):
        print(f"{o:10s} {n:14,d} {100 * n / te:5.1f}%  stalls {100 * st[o] / max(ts, 1):5.1f}%")


if __name__ == "__main__":
    main()
