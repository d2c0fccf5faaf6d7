"""Print the SASS of one kernel (substring match on the mangled name) from a .so."""
import subprocess, sys
so, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
cur, keep = None, []
for line in out.splitlines():
    if line.strip().startswith("Function :"):
        cur = line.strip().split(":", 1)[1].strip()
    if cur and pat in cur:
        keep.append(line)
print("\n".join(keep))
