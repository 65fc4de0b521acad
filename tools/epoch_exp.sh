python tools/gram_modes.py 5 0,2,1
RFD_GRAM_MODE=3 python tools/gram_once.py 5 2>&1 | sed -n 25,45p
for E in 16 64 256; do echo "EPOCH $E"; RFD_GRAM_EPOCH=$E python tools/gram_modes.py 5 0 ; RFD_GRAM_EPOCH=$E timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "config_parity or batched" 2>&1 | grep -E "cfg|passed|failed|\{" | head -8; done
