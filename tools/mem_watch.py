"""Dev: run __graft_entry__.smoke() with a watchdog that dumps every thread's
Python stack and exits when the process RSS passes a limit (GB, argv[1])."""
import faulthandler, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
LIMIT = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0

def rss_gb():
    with open("/proc/self/status") as f:
        for line in f:
            if line.startswith("VmRSS:"):
                return int(line.split()[1]) / 1e6
    return 0.0

def watch():
    while True:
        r = rss_gb()
        if r > LIMIT:
            print(f"RSS {r:.1f} GB > {LIMIT} GB", flush=True)
            faulthandler.dump_traceback(all_threads=True)
            os._exit(3)
        time.sleep(0.05)

threading.Thread(target=watch, daemon=True).start()
import __graft_entry__ as g
g.smoke()
print("smoke done, RSS", rss_gb())
