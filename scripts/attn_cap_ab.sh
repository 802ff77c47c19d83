# same-call A/B of the attention split cap (BST_ATTN_SPLIT_CAP) on the verify graph
for r in 1 2; do
  for n in 95 63; do
    for cap in 0 5 4 3; do
      echo -n "cap=$cap "; BST_ATTN_SPLIT_CAP=$cap python scripts/ablate_verify.py $n 2>&1 | tail -1
    done
  done
done
