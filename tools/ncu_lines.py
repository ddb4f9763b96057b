"""Aggregate an ncu `--page source --print-source=cuda,sass --csv` dump per CUDA source line."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    cur = "?"
    out = []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 8 and r[0] not in ("", "Line No") and r[0].isdigit():
            try:
                samples = int(r[4])
                inst = int(r[7])
            except ValueError:
                continue
            out.append((samples, inst, cur, int(r[0]), r[1][:90]))
    tot_s = sum(o[0] for o in out) or 1
    tot_i = sum(o[1] for o in out) or 1
    print(f"total samples {tot_s}  total warp-instructions {tot_i:,}")
    for key, name in ((0, "samples"), (1, "instructions")):
        print(f"--- top lines by {name}")
        for o in sorted(out, key=lambda x: -x[key])[:top]:
            print(f"{100*o[0]/tot_s:5.1f}% smp {100*o[1]/tot_i:5.1f}% ins  {o[2]}:{o[3]}  {o[4]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
