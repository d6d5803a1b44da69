#!/bin/bash
python scripts/k5dbg.py 2>&1 | tail -3
timeout 600 python -m pytest tests -q -m gpu -k "sensitiv or kmeans or dropin" 2>&1 | grep -E "passed|failed|Error|assert" | head -20
timeout 300 python scripts/time_k4k5.py 2>&1 | tail -12
