# e2e (host rays) streams x chunks sweep + a raw pinned H2D bandwidth probe
python - <<'PY' > gpurun_out/h2d_probe.txt 2>&1
import ctypes as C, numpy as np, sys, os
sys.path.insert(0, os.getcwd())
from paper_2210_04847_b200 import api
from paper_2210_04847_b200._lib import check
dev = api.Device(0); L = dev.lib
n = 184549376
p = C.c_void_p(); check(L.vmb_host_alloc(n, C.byref(p)))
d = dev.empty(n // 4, np.float32)
for _ in range(3): check(L.vmb_memcpy_h2d(dev.h, d.ptr, p.value, n))
dev.sync(); dev.record(0)
for _ in range(10): check(L.vmb_memcpy_h2d(dev.h, d.ptr, p.value, n))
dev.record(1); dev.sync()
ms = dev.elapsed_ms(0, 1) / 10
print("h2d 184 MB pinned:", round(ms, 3), "ms =", round(n / ms / 1e6, 1), "GB/s")
dev.record(0)
for _ in range(10): check(L.vmb_memcpy_d2h(dev.h, p.value, d.ptr, n))
dev.record(1); dev.sync()
ms = dev.elapsed_ms(0, 1) / 10
print("d2h 184 MB pinned:", round(ms, 3), "ms =", round(n / ms / 1e6, 1), "GB/s")
PY
cat gpurun_out/h2d_probe.txt
for cfg in "2 4" "2 8" "3 6" "4 8" "2 16" "3 3"; do
  set -- $cfg
  timeout 300 python bench.py --config1 0 --config2 0 --config3 0 --fields 0 --cpu-baseline 0 --phases 0 --steps 10 --e2e-streams $1 --e2e-chunks $2 > gpurun_out/e2e_$1_$2.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/e2e_$1_$2.json').read().strip().splitlines()[-1])
print('e2e S=$1 K=$2', round(d['e2e']['ms_per_step'],3), d['e2e']['matches_resident_outputs'], 'cam', round(d['e2e_camera']['ms_per_step'],3))"
done
