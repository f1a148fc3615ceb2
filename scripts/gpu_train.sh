set -x
timeout 600 python -m pytest tests/test_gpu_train.py -q -p no:cacheprovider --timeout 300 -x 2>&1 | tail -40
timeout 600 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider --timeout 300 2>&1 | tail -5
