# build paper_2104_01439_b200/libhh_$1.so from the working tree with extra nvcc flags ${@:2}
set -e
name=$1; shift
python - "$name" "$@" <<'PY'
import sys, subprocess
sys.path.insert(0, '/root/repo')
from paper_2104_01439_b200 import build as B
name, extra = sys.argv[1], sys.argv[2:]
cmd = [B.NVCC] + B.FLAGS + extra + ["-o", f"/root/repo/paper_2104_01439_b200/libhh_{name}.so"] + \
      ["/root/repo/paper_2104_01439_b200/csrc/" + s for s in B.SOURCES]
r = subprocess.run(cmd, capture_output=True, text=True)
print(f"libhh_{name}.so built" if r.returncode == 0 else r.stderr[-2000:])
PY
