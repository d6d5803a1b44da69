#!/bin/bash
timeout 900 python -m pytest tests -q -m gpu -k "hardening or store or kmeans or sensitiv" 2>&1 | tail -3
timeout 600 python scripts/time_retrieve.py > gpurun_out/retrieve.json 2>&1; cat gpurun_out/retrieve.json | tail -40
./scripts/ncu_r02.sh
