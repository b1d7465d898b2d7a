mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_product_kats.py tests/test_pipeline.py tests/test_gpu_parity.py tests/test_landmarks.py -m gpu -q -s -p no:cacheprovider > gpurun_out/r2_boundary.log 2>&1; echo "rc=$?" >> gpurun_out/r2_boundary.log
