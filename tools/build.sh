#!/bin/bash
# build the library from anywhere
cd "$(dirname "$0")/.." && python -c "from paper_1812_04315_b200 import _build; _build.build()" 2>&1 | grep -iE "error|warning" | head -20
