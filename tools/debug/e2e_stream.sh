set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or streaming" 2>&1 | tail -3
timeout 900 python bench.py --legs dense --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_dense_stream.json 2> gpurun_out/bench_dense_stream.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_dense_stream.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"])
PY
