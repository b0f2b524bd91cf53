for c in 1 2 4; do echo "ctas/SM=$c"; AJ_GJ_CTAS=$c AJ_VERBOSE=1 timeout 300 python scripts/prof_kernels.py 50 3 precond 1 2>&1 | grep "coarse"; done
