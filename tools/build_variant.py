"""Build a launch-configuration variant of the library (global engine only):
    python tools/build_variant.py THREADS MINB [extra nvcc flags...]
-> tools/variants/lib_t{THREADS}_b{MINB}.so (use with HCRAN_LIB=...)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1803_07772_b200 import build as B
t, b = int(sys.argv[1]), int(sys.argv[2])
extra = sys.argv[3:]
out = os.path.join(ROOT, 'tools', 'variants', f'lib_t{t}_b{b}.so')
os.makedirs(os.path.dirname(out), exist_ok=True)
cmd = [B.nvcc()] + B.NVCC_FLAGS + [f'-DHCRAN_THREADS={t}', f'-DHCRAN_MINB={b}', '-DHCRAN_NO_CLUSTER',
                                   '-I' + os.path.join(ROOT, 'include'), '-o', out] + extra + B.SOURCES
r = subprocess.run(cmd, capture_output=True, text=True)
open(out.replace('.so', '.log').replace('lib_', 'log_'), 'w').write(r.stderr)
print(out, r.returncode)
