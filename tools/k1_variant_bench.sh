for v in 3 0 1; do
  echo "variant=$v :: $(VS_K1_VARIANT=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --decoder-inputs 0 --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['single_batch']['value'], d['roofline']['frac'])")"
done
