#!/bin/bash
set -u
timeout 900 python -m pytest tests/test_slab_fuzz.py -q -p no:cacheprovider 2>&1 | tail -15
