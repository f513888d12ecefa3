timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_kernel -s 3 -c 1 -o gpurun_out/k1t_fw python tools/prof_k1.py 6400 42024 5 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_kernel -s 3 -c 1 -o gpurun_out/k1t_573 python tools/prof_k1.py 573 42024 5 > /dev/null 2>&1
