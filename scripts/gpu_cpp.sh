#!/bin/bash
# the C++ drivers (drop-in, multi-GPU build, device forward) on a B200
timeout 600 ./tests/cpp/_build/test_dropin | tail -2
timeout 900 ./tests/cpp/_build/test_build | tail -2
timeout 1800 ./tests/cpp/_build/test_forward --timing 2>&1 | tail -8
