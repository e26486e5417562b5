# narrow-band chase: cluster size and the no-dependency floor at small n
for v in "" "BSVD_CHASE_NC=3" "BSVD_CHASE_NC=2" "BSVD_CHASE_DIAG=48"; do echo "[$v]"; env $v python scripts/small_n.py 2>&1 | grep -v WRONG | head -2; done
