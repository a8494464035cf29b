"""Setup (tree + NNCA) time of lib variants at N=1M sphere (each lib in its own process, H2B_SETUP_VERBOSE on)."""
import os, subprocess, sys
here = os.path.dirname(os.path.abspath(__file__))
for lib in sys.argv[1:]:
    env = dict(os.environ, H2B_LIB=os.path.abspath(lib), H2B_SETUP_VERBOSE="1")
    r = subprocess.run([sys.executable, os.path.join(here, "setup_only.py"), "1048576", "2"], env=env,
                       capture_output=True, text=True)
    err = [l for l in r.stderr.splitlines() if l.startswith("[h2b]")]
    print(os.path.basename(lib), r.stdout.strip().splitlines()[-1:] or r.stderr[-400:], flush=True)
    for l in err[len(err) // 2:]:
        print("   ", l, flush=True)
