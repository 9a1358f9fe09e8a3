"""Opcode histogram per kernel of a cuobjdump -sass listing (stdin or file)."""
import re
import sys
from collections import Counter

txt = open(sys.argv[1]).read() if len(sys.argv) > 1 else sys.stdin.read()
for f in re.split(r'\n\s+Function : ', txt)[1:]:
    name = f.split('\n')[0]
    ops = re.findall(r'\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)', f)
    c = Counter(o if o.startswith(('VI', 'LD', 'ST')) else o.split('.')[0] for o in ops)
    print(name[:100], len(ops))
    print('   ', dict(c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 12)))
