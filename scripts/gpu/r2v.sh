for c in c2 c3 c4 c5; do timeout 900 python scripts/batch_paths.py $c 1 2 3 4 2>/dev/null | tail -1; done
