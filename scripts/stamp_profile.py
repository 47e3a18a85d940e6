"""Write the ncu --set full summary of a report into profiles/, stamped with the build stamp of
libfiber.so (sha256 of its SASS) so that bench.py uses its issue / SIMT / DRAM numbers only
for the build it was taken of.  Usage: stamp_profile.py <report.ncu-rep> <out.txt> [note]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from scripts.summarize_ncu import full  # noqa: E402

rep, out = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
full(rep, out + ".tmp")
body = open(out + ".tmp").read()
os.remove(out + ".tmp")
with open(out, "w") as f:
    f.write(f"# libfiber.so build stamp: {bench.lib_sha256()}\n")
    if note:
        f.write(f"# {note}\n")
    f.write(body)
print(open(out).read())
