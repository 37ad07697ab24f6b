"""Per-function SASS opcode histogram of a cubin/.so/executable.

usage: python tools/sass_mix.py <binary> [function-substring] [--loop]
"""
import collections
import re
import subprocess
import sys


def functions(binary):
    out = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            ins = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if ins:
                body.append((ins.group(2), line.strip()))
    if cur:
        yield cur, body


def main():
    binary = sys.argv[1]
    pat = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else ""
    for name, body in functions(binary):
        if pat not in name:
            continue
        hist = collections.Counter(op for op, _ in body)
        print(f"== {name}: {len(body)} instructions")
        for op, n in hist.most_common(25):
            print(f"   {n:6d} {op}")


if __name__ == "__main__":
    main()
