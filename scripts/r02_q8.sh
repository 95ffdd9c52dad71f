timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
DG_TRACE=1 timeout 300 python scripts/trace_tiles.py 2>&1 | grep -v "^ " | head -5
DG_TRACE=1 timeout 300 python scripts/trace_tiles.py --rows 1000000 2>&1 | grep -v "^ " | head -5
