O=gpurun_out/s4d; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_bands.py -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
TOFR_POOL_FRAC=0.4 timeout 900 python tools/c4_occupancy.py 16 8 16 > $O/occ.log 2>&1; tail -20 $O/occ.log
