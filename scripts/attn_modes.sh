# K3 key-major: cluster vs global merge at c=2K and 32K (BST_KT_MERGE forces a mode)
for m in auto global cluster; do
  BST_ATTN=kt BST_KT_MERGE=$m python scripts/bench_attention.py 2048 32768 | sed "s/^/$m /"
done
