# encrypt-ahead staging copies on their own copy stream: KV trace A/B, alternating
for e in "SPPIPE_SPEC_H2D=1" "X=1" "SPPIPE_SPEC_H2D=1" "X=1" "SPPIPE_SPEC_H2D=1" "X=1"; do
  env $e timeout 600 python tools/ab_switch.py none 2>&1 | grep '^{' | sed "s/^/$e /"
done
