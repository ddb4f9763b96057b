"""Stamp the DRAM traffic of the timed kernel from an ncu capture into
profiles/drive_kernel_traffic.json, with the hash of the kernel's sources, so bench.py
reports `roofline.traffic` only while the capture matches the kernel it times.

    python tools/ncu_traffic.py gpurun_out/prof_drive.ncu-rep
"""
import csv
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the production kernel's full source: drive_fast_kernel and the window math it inlines
KERNEL_SOURCES = ("paper_1604_04661_b200/csrc/sgns_fast.cuh", "paper_1604_04661_b200/csrc/sgns_device.cuh")


def kernel_source_hash(root=ROOT) -> str:
    h = hashlib.sha256()
    for rel in KERNEL_SOURCES:
        with open(os.path.join(root, rel), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def main(rep, out=os.path.join(ROOT, "profiles", "drive_kernel_traffic.json")):
    metrics = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread"
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", metrics],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}

    def val(name):
        v, u = float(vals[col[name]]), units[col[name]]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3,
                    "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(u, 1.0)

    commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True,
                            text=True).stdout.strip()
    rec = {"kernel": vals[col["Kernel Name"]] if "Kernel Name" in col else "drive_fast_kernel",
           "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
           "ncu_launch_ms_cold": val("gpu__time_duration.sum"),
           "registers": int(float(vals[col["launch__registers_per_thread"]])),
           "kernel_src_sha": kernel_source_hash(), "captured_at_commit": commit,
           "source": f"ncu --set full --clock-control none (profiles/run_ncu.sh), one warm launch "
                     f"of the default bench config; report {os.path.basename(rep)}"}
    with open(out, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
