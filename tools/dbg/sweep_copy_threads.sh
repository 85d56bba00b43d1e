for n in 2 4 8 12 15; do echo "threads=$n"; WF_HOST_COPY_THREADS=$n python tools/time_host.py 2>&1 | grep "daub4 numpy fuse 1 caller" | tail -2; done
