"""Aggregate ncu 'Instructions Executed' (warp-level) per CUDA source line.

  python tools/ncu_inst.py <report.ncu-rep> <object.o> <ncu-kernel-regex> <sass-function-substring> [top]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, obj, kname, fname = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
    page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kname}"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(page)))
    hdr, data = rows[1], rows[2:]
    ia, ii = hdr.index("Address"), hdr.index("Instructions Executed")
    base = int(data[0][ia], 16)
    inst = {int(r[ia], 16) - base: int(r[ii]) for r in data if r[ia].startswith("0x")}
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, check=True, capture_output=True)
        cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
        dis = subprocess.run(["nvdisasm", "-c", "--print-line-info", os.path.join(td, cub)],
                             capture_output=True, text=True).stdout
    infn, loc, line_of = False, None, {}
    for ln in dis.splitlines():
        if ln.startswith("//----") or ln.startswith("\t.section"):
            infn = fname in ln
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            loc = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]+)\*/", ln)
        if m and loc:
            line_of[int(m.group(1), 16)] = loc
    agg = collections.Counter()
    for off, c in inst.items():
        agg[line_of.get(off, "?")] += c
    tot = sum(agg.values()) or 1
    print(f"total warp instructions {tot}")
    for l, c in agg.most_common(top):
        print(f"{100 * c / tot:6.2f}% {c:14d} {l}")


if __name__ == "__main__":
    main()
