for R in 1 64 573; do for V in 4096 42024; do
 echo -n "R=$R V=$V flush: $(timeout 60 python tools/prof_k1.py $R $V 5 --legacy | tail -1 | sed 's/K1 ms per launch: \[[0-9.]*, \([0-9.]*\),.*GB\/s: \([0-9.]*\).*/\1 ms \2 GB\/s/') | noflush: "
 timeout 60 python tools/prof_k1.py $R $V 5 --legacy --noflush | tail -1 | sed 's/K1 ms per launch: \[[0-9.]*, \([0-9.]*\),.*GB\/s: \([0-9.]*\).*/\1 ms \2 GB\/s/'
done; done
