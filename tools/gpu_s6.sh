python tools/prof_kernels.py > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_random_search -s 256 -c 1 -o gpurun_out/prof_rs_lb python tools/prof_kernels.py > gpurun_out/ncu2.log 2>&1; tail -1 gpurun_out/ncu2.log
ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 1025 -c 1 -o gpurun_out/prof_prop_k7b python tools/prof_kernels.py > gpurun_out/ncu1.log 2>&1; tail -1 gpurun_out/ncu1.log
ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 1000 -c 1 -o gpurun_out/prof_prop_k1b python tools/prof_kernels.py > gpurun_out/ncu4.log 2>&1; tail -1 gpurun_out/ncu4.log
