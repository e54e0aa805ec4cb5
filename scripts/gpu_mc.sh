RF_DEBUG_LAUNCH=1 RF_K4_MC=1 timeout 120 python scripts/check_mc.py 2>&1 | grep "K4" | sort | uniq | head -5
