#!/bin/bash
# one line per gpurun_out/x_*.log bench result (experiment summaries)
for f in gpurun_out/x_*.log; do python -c "
import json,sys
l=[x for x in open('$f') if x.startswith('{')]
d=json.loads(l[-1]); r=d['roofline']; c=d['config']
print('%-28s'%'$f'[13:-4], '%8.1f us'%(d['ms_per_step']*1e3), 'kern %8.1f'%(r['kernel_ms']*1e3), '%5.1f%%'%c['pct_of_8tbs'], c['variant'], 'd16',c['d16'], 'tile',c['tile_nnz'])" 2>/dev/null || echo "$f fail: $(tail -1 $f)"; done
