#!/bin/bash
timeout 800 python -m pytest tests/test_gemm_gpu.py -x -q -m gpu -k "multicast" 2>&1 | tail -5
timeout 600 python -m pytest tests/test_copy_gpu.py -x -q -m gpu 2>&1 | tail -5
