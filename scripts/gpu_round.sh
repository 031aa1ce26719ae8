timeout 900 python -m pytest tests/test_gpu_build.py -x -q -m gpu 2>&1 | grep -E "^E|passed|failed|Error" | head
