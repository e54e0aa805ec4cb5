timeout 120 ./scripts/store_probe 131072 64
