# ncu --set full of the level-1 pass kernels as shipped (tools/prof_kernels.py on c5):
# k_propagate at PM iteration 7 (step 4, R41 skip active), k_random_search at iteration 7, k_reconstruct
set -e
python tools/prof_kernels.py > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 1025 -c 1 -o gpurun_out/prof_prop_k7 python tools/prof_kernels.py > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_random_search -s 256 -c 1 -o gpurun_out/prof_rs_k7 python tools/prof_kernels.py > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_reconstruct -s 27 -c 1 -o gpurun_out/prof_rec python tools/prof_kernels.py > gpurun_out/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 1000 -c 1 -o gpurun_out/prof_prop_k1 python tools/prof_kernels.py > gpurun_out/ncu4.log 2>&1
