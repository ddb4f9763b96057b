"""Top source lines per stall reason from an ncu cuda,sass source dump."""
import csv
import sys


def main(path, reasons=("stall_long_sb", "stall_short_sb", "stall_wait", "stall_branch_resolving"), top=8):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if len(r) > 10 and r[0] == "Line No")
    idx = {h: i for i, h in enumerate(hdr)}
    cur, out = None, []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 10 and r[0].isdigit():
            d = {}
            for c in reasons:
                try:
                    d[c] = int(r[idx[c]])
                except (ValueError, KeyError):
                    d[c] = 0
            out.append((cur, int(r[0]), r[1][:80], d))
    for c in reasons:
        tot = sum(o[3][c] for o in out) or 1
        print(f"=== {c} (total {tot})")
        for o in sorted(out, key=lambda o: -o[3][c])[:top]:
            print(f"  {100 * o[3][c] / tot:5.1f}% {o[0]}:{o[1]} {o[2]}")


if __name__ == "__main__":
    main(sys.argv[1])
