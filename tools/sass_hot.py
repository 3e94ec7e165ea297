"""Aggregate an ncu source page (--page source --csv --print-source sass) by opcode
and by address window: executed warp instructions and warp-stall samples."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ai, si, ei, wi = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    out = []
    base = None
    for r in rows[2:]:
        if len(r) <= ei or not r[ai].startswith("0x"):
            continue
        a = int(r[ai], 16)
        base = a if base is None else base
        op = r[si].strip().split()
        opc = op[0] if not op[0].startswith("@") else op[1]
        st = {hdr[i]: float(r[i] or 0) for i in stall_cols}
        out.append((a - base, opc, r[si].strip(), float(r[ei] or 0), float(r[wi] or 0), st))
    return out


if __name__ == "__main__":
    L = load(sys.argv[1])
    windows = [tuple(int(x, 16) for x in w.split(":")) for w in sys.argv[2:]]
    tot_e = sum(x[3] for x in L)
    tot_s = sum(x[4] for x in L)
    print("total executed warp inst %.4g, stall samples %.4g" % (tot_e, tot_s))
    byop = collections.defaultdict(lambda: [0.0, 0.0])
    for x in L:
        byop[x[1].split(".")[0]][0] += x[3]
        byop[x[1].split(".")[0]][1] += x[4]
    for k, (e, s) in sorted(byop.items(), key=lambda kv: -kv[1][0])[:20]:
        print("  %-10s exec %5.1f%%  samples %5.1f%%" % (k, 100 * e / tot_e, 100 * s / tot_s))
    stalls = collections.Counter()
    for x in L:
        stalls.update(x[5])
    print("stall reasons:", ", ".join("%s %.1f%%" % (k[6:], 100 * v / tot_s) for k, v in stalls.most_common(10)))
    # hottest 40-instruction windows
    W = 64
    seg = collections.defaultdict(lambda: [0.0, 0.0])
    for x in L:
        seg[x[0] // (16 * W)][0] += x[3]
        seg[x[0] // (16 * W)][1] += x[4]
    print("address windows (%d inst): exec%%, samples%%" % W)
    for k in sorted(seg):
        e, s = seg[k]
        if e / tot_e > 0.01 or s / tot_s > 0.01:
            print("  0x%05x  %5.1f%%  %5.1f%%" % (k * 16 * W, 100 * e / tot_e, 100 * s / tot_s))
