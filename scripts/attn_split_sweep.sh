# K3 split-count sweep in the 36-layer graph (scripts/attn_graph.py)
for sp in 0 14 16 17 19 20 24 36 37; do echo "splits=$sp"; SPLITS=$sp python scripts/attn_graph.py 32768 17 33; done
for sp in 0 1 2 3 4 5 6 8 12; do echo "splits=$sp"; SPLITS=$sp python scripts/attn_graph.py 2048 17 65 97 129; done
