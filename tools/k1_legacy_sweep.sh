for v in 3 1 0; do for pf in 0 1 2 4; do
 echo "v=$v pf=$pf :: $(VS_K1_VARIANT=$v VS_K1_PF=$pf timeout 100 python tools/prof_k1.py 6400 42024 5 bf16 --legacy | tail -1 | sed 's/.*GB/GB/') || $(VS_K1_VARIANT=$v VS_K1_PF=$pf timeout 100 python tools/prof_k1.py 573 42024 5 bf16 --legacy | tail -1 | sed 's/.*GB/GB/')"
done; done
