"""Aggregate ncu warp-stall samples per CUDA source line.

  python tools/ncu_lines.py <report.ncu-rep> <object.o> <ncu-kernel-regex> [top] [sass-function-substring]
  (NCU_LINES_COLUMN="Instructions Executed" aggregates another source-page column)

Exports the report's SASS source page, disassembles the kernel's cubin from
the object with line info (nvdisasm --print-line-info), maps every sampled
SASS address to the innermost file:line and prints the hottest lines.
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
    rep, obj, kname = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    fname = sys.argv[5] if len(sys.argv) > 5 else kname
    page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kname}"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(page)))
    hdr = rows[1]
    data = rows[2:]
    ia, iw = hdr.index("Address"), hdr.index(os.environ.get("NCU_LINES_COLUMN", "Warp Stall Sampling (All Samples)"))
    base = int(data[0][ia], 16)
    samples = {int(r[ia], 16) - base: int(float(r[iw] or 0)) for r in data if r[ia].startswith("0x")}
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, check=True,
                       capture_output=True)
        cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
        dis = subprocess.run(["nvdisasm", "-c", "--print-line-info", os.path.join(td, cub)],
                             capture_output=True, text=True).stdout
    infn, loc = False, None
    line_of = {}
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
    for off, s in samples.items():
        agg[line_of.get(off, "?")] += s
    tot = sum(agg.values()) or 1
    print(f"total samples {tot}")
    for loc, s in agg.most_common(top):
        print(f"{100 * s / tot:6.2f}%  {loc}")


if __name__ == "__main__":
    main()
