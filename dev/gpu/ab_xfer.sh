cd $GRAFT_REPO_ROOT
for cfg in "8 8" "16 8" "16 4" "32 4" "8 16"; do set -- $cfg
OPCFE_XFER_SLOTS=$1 OPCFE_XFER_CHUNK_MB=$2 python dev/dropin_profile.py 2>&1 | grep "strict:" | tail -1 | sed "s/^/slots=$1 chunk=$2 /"
done
