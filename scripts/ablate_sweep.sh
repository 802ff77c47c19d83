for n in 31 63 127 255; do
  for a in "" attn resid swiglu rope "attn,resid,swiglu,rope"; do
    BST_ABLATE=$a python scripts/ablate_verify.py $n 2>&1 | tail -1
  done
done
