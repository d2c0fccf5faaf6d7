"""Registers / spills per K1 instantiation from a ptxas -v report."""
import re, sys
txt = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2602_22421_b200/ptxas_report.txt").read()
pat = re.compile(r"Compiling entry function '(_ZN5spfom\w+)' for 'sm_100a'\n(?:ptxas info\s+: Function properties for \S+\n)?\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\nptxas info\s+: Used (\d+) registers")
filt = sys.argv[2] if len(sys.argv) > 2 else "k_primal"
for m in pat.finditer(txt):
    name = m.group(1)
    if filt not in name:
        continue
    short = re.sub(r"EEEvNS_8DevState.*", "", re.sub(r"_ZN5spfom\d+", "", name)).replace("ILi", "<").replace("ELi", ",").replace("ELb", ",b").replace("ILb", "<b")
    print(f"{short:40s} regs {m.group(5):>3s} spill st {m.group(3):>4s} ld {m.group(4):>4s}")
