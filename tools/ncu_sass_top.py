"""Top SASS instructions of an ncu source page (csv, --print-source sass) by
warp-stall samples, with source line (nvdisasm -g) and the dominant stall reasons.
    python tools/ncu_sass_top.py <sass_page.csv> <nvdisasm_g.txt> <mangled kernel name> [N]"""
import collections
import csv
import re
import sys


def main(page, dis, fn, n=40):
    txt = open(dis).read().split("\n")
    start = next(i for i, l in enumerate(txt) if l.startswith(".text." + fn + ":"))
    addr2 = {}
    cur = None
    for l in txt[start + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r'//## File "(.*?)", line (\d+)', l)
        if m:
            cur = "%s:%s" % (m.group(1).split("/")[-1], m.group(2))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m and cur is not None:
            addr2[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(page)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r)
    h = rows[hi]
    ia, iw, isrc = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    ir = [h.index(c) for c in reasons]
    data = []
    base = None
    for r in rows[hi + 1:]:
        try:
            a = int(r[ia], 16)
            w = float(r[iw] or 0)
        except (ValueError, IndexError):
            continue
        if base is None:
            base = a
        rs = {reasons[k][6:]: float(r[ir[k]] or 0) for k in range(len(ir))}
        data.append((w, a - base, r[isrc].strip(), rs))
    tot = sum(d[0] for d in data)
    byline = collections.Counter()
    for w, off, src, rs in data:
        byline[addr2.get(off, "?")] += w
    print("total samples", tot)
    for w, off, src, rs in sorted(data, key=lambda d: -d[0])[:n]:
        top = sorted(rs.items(), key=lambda kv: -kv[1])[:3]
        print("%5.1f%% %05x %-18s %-46s %s" % (100 * w / tot, off, addr2.get(off, "?"), src[:46],
                                               " ".join("%s=%d" % kv for kv in top if kv[1] > 0)))
    print("--- by source line")
    for k, w in byline.most_common(n):
        print("%5.1f%% %s" % (100 * w / tot, k))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
