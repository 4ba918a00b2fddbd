#!/bin/bash
# IPC transport + CLI boundary tests, then a quick per-preset timing
OUT=gpurun_out/${TAG:-ipc}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_decomp_ipc.py tests/test_cli.py -m gpu -q -p no:cacheprovider -x > $OUT/pytest.log 2>&1
tail -15 $OUT/pytest.log
