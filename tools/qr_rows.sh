# NENMF_QR_ROWS sweep: QR of a 10^4 x 30 panel and the cfg2 RSI vs rows per Gram-partial CTA (development aid)
for r in 256 512 1024 2048; do
  echo "NENMF_QR_ROWS=$r"; NENMF_QR_ROWS=$r python tools/qr_bench.py 30 10000; NENMF_QR_ROWS=$r python tools/probe_cfg.py 2 1 2>&1 | grep RSI
done
