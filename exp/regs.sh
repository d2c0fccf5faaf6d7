#!/usr/bin/env bash
# ptxas registers / spills per K1 stream instantiation for a set of -D flags
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v "$@" -I include -c -o /tmp/regs_t.o paper_2602_22421_b200/csrc/spfom.cu 2>&1 | \
python3 -c "
import sys,re,subprocess
name=None
for l in sys.stdin:
    m=re.search(r\"Compiling entry function '(\S+)'\",l)
    if m: name=m.group(1); continue
    if name and 'spill' in l: sp=re.search(r'(\d+) bytes spill stores',l).group(1)
    if name and 'Used' in l and 'registers' in l:
        if 'k_primal' in name:
            d=subprocess.run(['c++filt',name],capture_output=True,text=True).stdout.strip().replace('spfom::','').split('(')[0]
            print(f'{d:45s} regs {re.search(r\"Used (\d+)\",l).group(1):>4s} spill {sp}')
        name=None
"
