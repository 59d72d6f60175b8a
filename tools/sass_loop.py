"""Instruction mix of an address range of a cuobjdump -sass listing.
usage: python tools/sass_loop.py file.sass start_hex end_hex [steps]"""
import re, sys, collections
f, a, b = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
c = collections.Counter()
for ln in open(f):
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', ln)
    if m and a <= int(m.group(1), 16) <= b:
        t = re.sub(r'^@!?U?P\w+\s+', '', m.group(2).strip())
        c[t.split()[0]] += 1
print(sum(c.values()), 'instructions', sum(c.values()) / steps, 'per step')
for k, v in c.most_common(45):
    print(v, k)
