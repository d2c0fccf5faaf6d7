"""K1 variants on one config: for each library (SPFOM_LIB-style paths given on
the command line) time K1 in two windows -- the transient (iterations
W0..W0+n) and the steady state (iterations S0..S0+n) -- with the split-graph
timed stepping bench.py uses.  Each library runs in its own subprocess (one
libspfom per process).  CFG=huge|medium|multi (default huge)."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ".")
    import bench  # noqa: E402
    from paper_2602_22421_b200 import Params, Solver  # noqa: E402
    cfg = os.environ.get("CFG", "huge")
    inst = bench.load_instance(cfg, "/tmp/spfom_cache")
    pad = int(os.environ.get("PAD_GIB", "0"))
    s = Solver(inst, Params.converge(), device="cuda:0", workspace_offset_bytes=pad << 30)
    if os.environ.get("TOUCH"):
        s.residuals()        # load the residual kernels now (lazy module loading)
        s.recover_timed()
    out = {}
    n = int(os.environ.get("N", "100"))
    for name, start in (("early", 5), ("late", int(os.environ.get("LATE", "1500"))),
                        ("late2", int(os.environ.get("LATE", "1500")) + 500)):
        s.step(start - s.iteration)
        r0 = s.residuals()
        k1, tot = s.step_timed(n)
        r1 = s.residuals()
        out[name] = dict(k1_ms=round(k1 / n, 5), step_ms=round(tot / n, 5),
                         passes=round((r1["newton_passes"] - r0["newton_passes"]) / (n * inst.m), 3))
    out["fail"] = s.residuals()["newton_failures"]
    print(json.dumps(out))
    sys.exit(0)

for lib in sys.argv[1:]:
    env = dict(os.environ, SPFOM_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-600:]
    print(f"{os.path.basename(lib):24s} {line}", flush=True)
    if os.environ.get("SHOW_BINS"):      # -DSPFOM_DIAG_BIN_SMS libraries: the bins' weights and SM shares
        print("".join(sorted(set(l + "\n" for l in r.stderr.splitlines() if l.startswith("[spfom] bin")))), end="", flush=True)
