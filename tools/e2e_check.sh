for i in 1 2; do python bench.py --no-cpu-baseline --steps 2000 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step']*1e3,2), round(d['e2e']['value']/1e6,3))"; done
timeout 300 python -m pytest tests/test_data_ingest.py -q -m gpu 2>&1 | tail -1
