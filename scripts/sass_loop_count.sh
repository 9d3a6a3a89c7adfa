#!/bin/bash
# count SASS instructions in K4's hot loop (from the first MUFU.EX2 block's loop head to its back-edge)
cd /root/repo/paper_2604_25459_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -cubin -o /tmp/k4.cubin k4_composite.cu || exit 1
cuobjdump -sass -fun "$1" /tmp/k4.cubin > /tmp/k4.sass
python3 - <<'PY'
import re
ins=[l for l in open('/tmp/k4.sass').read().splitlines() if re.match(r'\s+/\*[0-9a-f]+\*/',l)]
txt=[re.sub(r'\s+',' ',l.split(';')[0]).strip() for l in ins]
# loop over set records: from LDS.U8 (wlist) to the backward branch after the last MUFU region
first=[i for i,t in enumerate(txt) if 'LDS.U8' in t][0]
mu=[i for i,t in enumerate(txt) if 'MUFU.EX2' in t]
back=[i for i,t in enumerate(txt) if i>mu[-1] and 'BRA' in t][0]
print('hot region instructions:', back-first+1, ' MUFU count:', len(mu))
PY
