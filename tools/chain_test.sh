#!/bin/bash
# correctness + timing of the dataflow lookahead chain (TFB_CHAIN_DATAFLOW=1)
export TFB_CHAIN_DATAFLOW=1
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_zero_pivot.py tests/test_gpu_races.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
unset TFB_CHAIN_DATAFLOW
bash tools/ab_env.sh cfg5 TFB_CHAIN_DATAFLOW 0 1
bash tools/ab_env.sh cfg4 TFB_CHAIN_DATAFLOW 0 1
