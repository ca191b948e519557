timeout 2400 python tools/config5.py 1250 512 67108864 > gpurun_out/r2_config5_share_w4096geom.json 2> gpurun_out/r2_config5_share.err; echo "rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r2_config5_share_w4096geom.json').read()); d.pop('per_chunk_bits_per_base'); print(d)"
