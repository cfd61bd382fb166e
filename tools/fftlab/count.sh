#!/bin/bash
# count SASS instructions per probe kernel, by class
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -cubin -o /tmp/wfft_probe.cubin wfft_probe.cu || exit 1
cuobjdump -sass /tmp/wfft_probe.cubin > /tmp/wfft_probe.sass
python3 - <<'PY'
import re, collections
cur=None; c=collections.defaultdict(collections.Counter)
for line in open('/tmp/wfft_probe.sass'):
    m=re.search(r'Function : (\S+)', line)
    if m: cur=m.group(1); continue
    m=re.match(r'\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9]*)', line)
    if m and cur: c[cur][m.group(1)]+=1
for k,v in c.items():
    tot=sum(v.values()); dp=v['DADD']+v['DMUL']+v['DFMA']
    print(k[-40:], 'total', tot, 'DP', dp, ' '.join(f'{o}:{n}' for o,n in v.most_common(14)))
PY
