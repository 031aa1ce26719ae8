timeout 900 python -m pytest tests/test_gpu_api.py -x -q -m gpu 2>&1 | grep -E "^E|Error|error|passed|failed|test_" | head -20
