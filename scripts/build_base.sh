# build libhh_A.so (A/B baseline) from git revision $1 (default HEAD)
set -e
rev=${1:-HEAD}
rm -rf /tmp/base && mkdir -p /tmp/base
git archive $rev paper_2104_01439_b200/csrc include | tar -x -C /tmp/base
python - <<'PY'
import sys, subprocess
sys.path.insert(0, '/root/repo')
from paper_2104_01439_b200 import build as B
cmd = [B.NVCC] + B.FLAGS + ["-o", "/root/repo/paper_2104_01439_b200/libhh_A.so"] + \
      ["/tmp/base/paper_2104_01439_b200/csrc/" + s for s in B.SOURCES]
r = subprocess.run(cmd, capture_output=True, text=True)
print("libhh_A.so built" if r.returncode == 0 else r.stderr[-2000:])
PY
