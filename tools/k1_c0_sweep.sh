for c in 0.05 0.2 0.5 1 2 4; do
  echo "c0=$c :: $(VS_K1_C0=$c timeout 60 python tools/prof_k1.py 573 42024 5 | tail -1 | sed 's/.*GB/GB/') || nf $(VS_K1_C0=$c timeout 60 python tools/prof_k1.py 573 42024 5 bf16 --noflush | tail -1 | sed 's/.*GB/GB/') || 1500 $(VS_K1_C0=$c timeout 60 python tools/prof_k1.py 1500 42024 5 | tail -1 | sed 's/.*GB/GB/') || 6400 $(VS_K1_C0=$c timeout 60 python tools/prof_k1.py 6400 42024 5 | tail -1 | sed 's/.*GB/GB/') || 64 $(VS_K1_C0=$c timeout 60 python tools/prof_k1.py 64 42024 5 | tail -1 | sed 's/.*GB/GB/')"
done
for c in 0.05 0.5 2; do echo "bench c0=$c :: $(VS_K1_C0=$c timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decoder-inputs 0 --e2e-steps 1 --streams 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['roofline']['frac'])")"; done
