"""Per-basic-block instruction counts of one kernel in an ncu report
(development tool).   python tools/ncu_hot.py report.ncu-rep kernel_regex [min_share]"""
import csv
import io
import subprocess
import sys


def main():
    rep, pat = sys.argv[1], sys.argv[2]
    share = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
    import re
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "Kernel Name" and re.search(pat, r[1]))
    rows = rows[start:]
    h = rows[1]
    ie, src = h.index("Instructions Executed"), h.index("Source")
    st = h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        if len(r) > ie and r[ie].isdigit():
            data.append((int(r[ie]), int(r[st] or 0), r[0][-5:], r[src].strip()))
        elif r and "Kernel Name" in r[0]:
            break
    tot = sum(d[0] for d in data)
    print("instructions", tot, "stall samples", sum(d[1] for d in data))
    groups = []
    for c, s, a, t in data:
        if groups and groups[-1][0] == c:
            g = groups[-1]
            g[1] += 1
            g[4] += s
            g[5].append(t)
        else:
            groups.append([c, 1, a, t, s, [t]])
    for c, n, a, t, s, body in groups:
        if c * n >= share * tot:
            print("%10d x %3d = %10d  stalls %6d  @%s  %s" % (c, n, c * n, s, a, " | ".join(x[:28] for x in body[:6])))


if __name__ == "__main__":
    main()
