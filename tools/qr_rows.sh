for r in 256 512 1024 2048; do
  echo "NENMF_QR_ROWS=$r"; NENMF_QR_ROWS=$r python tools/qr_bench.py 30 10000; NENMF_QR_ROWS=$r python tools/probe_cfg.py 2 1 2>&1 | grep RSI
done
