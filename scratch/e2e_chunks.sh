for c in 256 512 1024 2048 4096; do FT_STREAM_CHUNK=$c python scratch/e2e.py 2>&1 | grep streamed | sed "s/^/C=$c /"; done
