"""Map an ncu SASS source page (csv) of one kernel onto CUDA source lines via
nvdisasm -g line info, and print the lines with the most warp-stall samples.
    python tools/ncu_src_hotspots.py <sass_page.csv> <nvdisasm_g.txt> <mangled kernel name> [N]"""
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
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m and cur is not None:
            addr2[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(page)))
    h = rows[1]
    ia, iw, ie = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    base = None
    agg, ins = collections.Counter(), collections.Counter()
    tot = 0.0
    for r in rows[2:]:
        try:
            a = int(r[ia], 16)
        except (ValueError, IndexError):
            continue
        base = a if base is None else base
        w = float(r[iw] or 0)
        tot += w
        key = addr2.get(a - base, ("?", 0))
        agg[key] += w
        ins[key] += float(r[ie] or 0)
    srcs = {}
    for (f, ln), w in agg.most_common(n):
        text = ""
        if f.endswith((".cu", ".cuh")):
            try:
                srcs.setdefault(f, open("paper_2206_03410_b200/csrc/" + f).read().split("\n"))
                text = srcs[f][ln - 1].strip()[:90]
            except OSError:
                pass
        print(f"{w / tot * 100:5.1f}%  inst {ins[(f, ln)]:11.0f}  {f}:{ln}  {text}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
