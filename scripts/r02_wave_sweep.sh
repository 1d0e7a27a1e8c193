set -x
python -m pytest tests -m gpu -q -x 2>&1 | tail -15
for W in 49152 16384 32768 100000 300000; do
  FALCON_ENC_WAVE_CHUNKS=$W python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('W=$W', round(d['value'],1), 'enc', round(r['encode_kernel_ms'],4), 'dec', round(r['decode_kernel_ms'],4), 'step', round(d['ms_per_step'],4))"
done
