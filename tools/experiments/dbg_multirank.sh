python -m pytest tests/test_multirank.py -m gpu -q -x 2>&1 | tail -3
CUDA_LAUNCH_BLOCKING=1 python -m pytest tests/test_multirank.py -m gpu -q 2>&1 | tail -3
python -m pytest tests/test_multirank.py -m gpu -q -k "c1-2" 2>&1 | tail -3
