# A/B of the host-output receiver-chunk schedules (capi.cu kSched)
for rep in 1 2; do for s in 0 2 3 6; do RXGS_E2E_SCHED=$s python scripts/probe_e2e_sched.py 2>&1 | tail -1; done; done
