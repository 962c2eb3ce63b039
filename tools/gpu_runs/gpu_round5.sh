set -x
python -m pytest tests/test_gpu_parity.py -x -q -k GRAMSCHM 2>&1 | tail -5
python tools/variant_report.py --out gpurun_out/variant_report_gs.json --benches GRAMSCHM --skip-ms 30 2>&1 | tail -3
python - <<'PY'
import json; r=json.load(open('gpurun_out/variant_report_gs.json'))['benches']['GRAMSCHM']['all_ms']
print({k: round(v,3) for k,v in r.items() if not k.startswith('stage=0') or 'unroll=0' in k})
PY
