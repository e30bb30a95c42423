# same-box A/B of the level-kernel forms: register-staged tiles vs the streaming-march chassis
for m in "" "--march"; do
  for spec in "16384 8192 0" "8192 16384 0" "1024 65536 1"; do
    set -- $spec
    python profiles/kernel_probe.py --time --n-el $1 --n-t $2 --dir $3 $m --only sweep,restrict,restrict_zero,prolong_sweep_zero,norm_sweep,prolong_sweep
  done
done
