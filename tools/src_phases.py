"""Attribute a kernel's executed instructions and stall samples to source
phases: SASS rows in address order, each credited to the most recent line of
the kernel's own file (inlined helpers from other headers inherit the caller
line). Usage: src_phases.py <cuda,sass csv> <sass csv> <file> <ranges>
where ranges = "name:lo-hi,name:lo-hi,..." (line numbers of <file>)."""
import csv
import sys


def main(combined, sass, fname, ranges):
    amap, fp, cur = {}, None, None
    for r in csv.reader(open(combined)):
        if r and r[0] == "File Path":
            fp = r[1].split("/")[-1]
            continue
        if not r or r[0] in ("Function Name", "Line No"):
            continue
        if r[0] != "":
            cur = (fp, int(r[0]))
        elif len(r) > 2 and r[2].startswith("0x"):
            amap[r[2]] = cur
    ph = [(n, int(a), int(b)) for n, ab in (x.split(":") for x in ranges.split(",")) for a, b in [ab.split("-")]]
    agg, last = {}, None
    tot_i = tot_s = 0
    for r in csv.reader(open(sass)):
        if len(r) < 8 or not r[0].startswith("0x"):
            continue
        ie = int(r[5]) if r[5].isdigit() else 0
        st = int(r[2]) if r[2].isdigit() else 0
        src = amap.get(r[0])
        if src and src[0] == fname:
            last = src[1]
        name = "other"
        if last is not None:
            for n, a, b in ph:
                if a <= last <= b:
                    name = n
                    break
        a = agg.setdefault(name, [0, 0])
        a[0] += ie
        a[1] += st
        tot_i += ie
        tot_s += st
    print(f"| phase | warp instructions | share | stall samples | share |")
    print("|---|---|---|---|---|")
    for n, _, _ in ph + [("other", 0, 0)]:
        if n in agg:
            i, s = agg[n]
            print(f"| {n} | {i} | {100 * i / tot_i:.1f}% | {s} | {100 * s / max(tot_s, 1):.1f}% |")
    print(f"| total | {tot_i} | | {tot_s} | |")


if __name__ == "__main__":
    main(*sys.argv[1:5])
