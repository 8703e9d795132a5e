#!/usr/bin/env bash
# build the native libraries from anywhere
cd "$(dirname "$0")/.." && python -c "from paper_2602_02204_b200 import build as b; b.build()"
