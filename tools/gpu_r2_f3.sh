mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_pipeline.py tests/test_landmarks.py -m gpu -q -s -p no:cacheprovider > gpurun_out/r2_f3.log 2>&1; echo "rc=$?" >> gpurun_out/r2_f3.log
