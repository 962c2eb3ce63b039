set -x
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
python tools/variant_report.py --out gpurun_out/variant_report_dense.json --benches GEMM 2MM 3MM SYRK SYR2K CORR COVAR 2>&1 | tail -9
python - <<'PY'
import sys, statistics
sys.path.insert(0, '.')
from paper_1810_10496_b200.backend.b200 import B200Backend, family
be = B200Backend(device=0)
fam = family('GRAMSCHM')
for key in ('stage=1', 'stage=2,vec=0', 'stage=2,vec=1'):
    v = next(i for i in range(len(fam.knobs)) if fam.key(i) == key)
    ws = be.workspace('GRAMSCHM', (2048, 2048), True, -1)
    ws.run(v, samples=1, restore=True)
    print('GRAMSCHM', key, [round(x, 3) for x in ws.run(v, samples=3, restore=True, flush=True)])
PY
