for c in 4 16 64; do RD_HOST_CHUNK_MB=$c python tools/e2e_time.py; done
