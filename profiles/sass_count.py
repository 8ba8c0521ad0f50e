"""Static SASS opcode counts per kernel of an object/library (cuobjdump -sass).
usage: python profiles/sass_count.py build/ssm_pw.o [kernel-substring]"""
import collections
import re
import subprocess
import sys


def main(path, sub=""):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, counts = None, collections.defaultdict(collections.Counter)
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m and cur:
            counts[cur][m.group(2)] += 1
    for f, c in counts.items():
        if sub in f:
            print(f, sum(c.values()), c.most_common(12))


if __name__ == "__main__":
    main(*sys.argv[1:])
