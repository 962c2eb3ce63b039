# tcgen05 contraction bottleneck split: time 2MM/SYRK stage=2 with parts of the
# pipeline disabled (PF_TC_DIAG: 1 no lo split, 2 no MMAs, 4 no loads) for the
# single-CTA and CTA-pair kernels.  Outputs are wrong in diag modes (timing only).
for pair in 1 0; do
  for diag in 0 1 2 4 5 6 3; do
    echo "pair=$pair diag=$diag $(PF_TC_PAIR=$pair PF_TC_DIAG=$diag timeout 120 python tools/profile_kernels.py 2MM 2048,2048,2048,2048 stage=2 10 2>&1 | tail -1)"
  done
done
