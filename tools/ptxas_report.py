#!/usr/bin/env python
"""Per-kernel registers / spills / stack from the build's ptxas -v logs."""
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(pattern=""):
    for log in sorted(glob.glob(os.path.join(ROOT, "build", "native", "*.o.log"))):
        name = None
        for line in open(log):
            m = re.search(r"Compiling entry function '([^']+)'", line)
            if m:
                name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
                stack = spill = None
            m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
            if m:
                stack, spill = int(m.group(1)), (int(m.group(2)), int(m.group(3)))
            m = re.search(r"Used (\d+) registers", line)
            if m and name:
                if pattern in name:
                    short = re.sub(r"\(.*", "", name)
                    print(f"{short:60s} regs={m.group(1):>4s} stack={stack:>4d} spill={spill}")
                name = None


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "")
