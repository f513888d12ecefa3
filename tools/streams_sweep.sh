timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "concurrent or decode" 2>&1 | tail -2
for S in ${SWEEP:-2 3 4 6}; do
  echo "S=$S :: $(timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --decoder-inputs 0 --streams $S 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['gpu_launches'])")"
done
