#!/bin/bash
python -m pytest tests/test_gpu_parity.py -q -x -k "bit_granular or packed_encoder" 2>&1 | tail -3
python tools/exp/enc_bits.py
