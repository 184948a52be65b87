for r in 1 2; do
for v in "X=1" "SRPB_OTF_NFAST=1" "SRPB_OTF_LOCKSTEP=1" "SRPB_TC_NMAX=128"; do
  echo "$v $(env $v timeout 300 python tools/c4_probe.py --frames 640 --conv-cands 0 --reps 2 2>&1 | grep -E 'maps=True' | sed 's/.*J=600000: //')"
done; done
