# KV trace under crypto SM budgets (ReplayConfig.crypto_sms)
for e in "X=1" "AB_CRYPTO_SMS=16" "AB_CRYPTO_SMS=32" "AB_CRYPTO_SMS=48" "AB_CRYPTO_SMS=64"; do
  env $e timeout 600 python tools/ab_switch.py none 2>&1 | tail -1 | sed "s/^/$e /"
done
