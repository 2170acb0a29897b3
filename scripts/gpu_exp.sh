timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings -k "list_triangles or golden" 2>&1 | tail -3
