"""A/B per-layer comparison of two op_profile logs (profiling helper)."""
import re
import sys


def parse(f):
    out, hdr = [], []
    for line in open(f):
        if "exec p50" in line:
            hdr.append(line.strip())
        m = re.match(r"\s*(\d+) (\w+)\s+(\d+)->\s*(\d+) k(\d) s(\d) @\s*(\d+) .*?\+\s*([\d.]+) us", line)
        if m:
            out.append((m.group(2), int(m.group(3)), int(m.group(4)), int(m.group(5)), int(m.group(7)),
                        float(m.group(8))))
    return out, hdr


a, ha = parse(sys.argv[1])
b, hb = parse(sys.argv[2])
print("A:", *ha, sep="\n  ")
print("B:", *hb, sep="\n  ")
a = [x for x in a if x[0] != "maxpool"]
b = [x for x in b if x[0] != "maxpool"]
for x, y in zip(a, b):
    flag = " <<" if y[5] > x[5] * 1.1 + 0.5 else (" >>" if y[5] < x[5] * 0.9 - 0.5 else "")
    print(f"{x[0]:7s} {x[1]:5d}->{x[2]:5d} k{x[3]} @{x[4]:3d}  A {x[5]:6.1f}  B {y[5]:6.1f}{flag}")
