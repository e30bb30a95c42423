#!/bin/bash
# Same-box A/B of compile-time variants built by profiles/ab_build.py into ab/<name>/:
#   bash profiles/ab_variants.sh default <name> ...      (default = the in-tree build)
for v in "$@"; do
  if [ "$v" = default ]; then unset STMG_LIB_PATH; else export STMG_LIB_PATH=ab/$v/libstmg_b200.so; fi
  echo "== $v"; python profiles/kernel_probe.py --time; python profiles/fusion_ab.py --config cfg2 --flags 1 --solves 3 --profile 0
done
