#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "many_units" 2>&1 | tail -3
