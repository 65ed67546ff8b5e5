# A/B of host-pipeline variants (development aid): e2e_probe under env knobs
for rep in 1 2; do
UFPGD_E2E_PIPE=1 python tools/e2e_probe.py
for r in none up down both; do echo ramp=$r; UFPGD_HOST_RAMP=$r python tools/e2e_probe.py; done
done
UFPGD_HOST_RAMP=both python tools/host_timeline.py
python -m pytest -q tests/test_gpu_edge.py tests/test_gpu_parity.py -k "host" -p no:cacheprovider 2>&1 | tail -2
