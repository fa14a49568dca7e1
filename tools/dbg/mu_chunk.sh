for c in 2 4 6 8; do
  ST_MU_CHUNK=$c python bench.py --quick 2>/dev/null > gpurun_out/q.json
  python -c "import json; d=json.load(open('gpurun_out/q.json')); print('chunk', $c, round(d['value'],1), round(d['stage_ms']['mu_raster_side_stream'],3), round(d['stage_ms']['mu_wait'],3))"
done
