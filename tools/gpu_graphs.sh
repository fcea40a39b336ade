# CUDA-graph check: parity tests of the driver, then the config table with graphs on and off
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "graph or pipeline" > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
python tools/config_table.py > gpurun_out/config_table_graphs.log 2>&1
VINP_NO_GRAPHS=1 python tools/config_table.py > gpurun_out/config_table_eager.log 2>&1
