PBH_PHASES=1 timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import paper_1908_09378_b200 as P
from paper_1908_09378_b200 import gen
g = gen.grid(1024, 1024, 1)
ctx = P.SsspContext(g, max_sources=1, mode='threshold')
ms = ctx.run([0]); r = ctx.fetch(0, settled=False); print('ms', ms, 'batches', r.rounds)
" 2>&1 | tail -3
