bash tools/gjob_tests.sh
timeout 600 python tools/stage_sensitivity.py C2 2>&1 | grep -v Warn
timeout 900 python tools/stage_sensitivity.py C4 2>&1 | grep -v Warn
