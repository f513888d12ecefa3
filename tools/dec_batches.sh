for b in 1 2 3; do
timeout 900 python -c "
import sys, json
sys.argv=['bench']
import bench
w = bench.WORKLOADS['wmt19_k50']
r = bench.decoder_leg(w, 2000, batches=$b)
print($b, r['value'], r['ms_per_timestep'], r['timesteps'])
"
done
