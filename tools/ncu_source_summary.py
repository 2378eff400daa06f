"""Summarise an ncu `--page source --csv --print-source=cuda,sass` dump:
executed warp instructions and stall samples per SASS opcode and per source
line (file:line). Usage: python tools/ncu_source_summary.py dump.csv [top]"""
import collections
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path)))
by_op = collections.Counter()
stall_op = collections.Counter()
by_line = collections.Counter()
stall_line = collections.Counter()
fname = "?"
cur_line = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9:
        continue
    if r[0]:
        cur_line = "%s:%s" % (fname, r[0])
    sass = r[3].strip()
    # with --print-source=cuda,sass every CUDA source line also has an
    # aggregate row ("-" in the SASS column) repeating the counts of the SASS
    # rows below it: counting it too doubled every total (round-1 summaries)
    if not sass or sass == "-" or not r[2] or r[2] == "...":
        continue
    op = sass.split()[0] if not sass.startswith("@") else sass.split()[1]
    op = op.split(".")[0]
    def num(v):
        try:
            return float(v)
        except ValueError:
            return 0.0
    ex = num(r[7])
    st = num(r[4])
    by_op[op] += ex
    stall_op[op] += st
    by_line[cur_line] += ex
    stall_line[cur_line] += st
tot = sum(by_op.values())
tst = sum(stall_op.values())
print("total warp instructions %.4g, stall samples %.4g" % (tot, tst))
print("%-12s %10s %7s %7s" % ("opcode", "inst", "%inst", "%stall"))
for op, v in by_op.most_common(top):
    print("%-12s %10.4g %6.1f%% %6.1f%%" % (op, v, 100 * v / tot, 100 * stall_op[op] / tst))
print()
print("%-28s %10s %7s %7s" % ("line", "inst", "%inst", "%stall"))
for ln, v in sorted(by_line.items(), key=lambda kv: -stall_line[kv[0]])[:top]:
    print("%-28s %10.4g %6.1f%% %6.1f%%" % (ln, v, 100 * v / tot, 100 * stall_line[ln] / tst))
print()
print("%-28s %10s %7s %7s   (by instructions)" % ("line", "inst", "%inst", "%stall"))
for ln, v in by_line.most_common(top):
    print("%-28s %10.4g %6.1f%% %6.1f%%" % (ln, v, 100 * v / tot, 100 * stall_line[ln] / tst))
