"""Debug driver: PipeFusion stage processes on one GPU, one case, verbose, short timeout."""
import json, multiprocessing as mp, os, sys, tempfile, socket
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import _peer_worker

if __name__ == "__main__":
    world = int(sys.argv[1]); ci = [int(x) for x in sys.argv[2].split(",")]
    from tests.test_gpu_peer import PF_CASES
    cases = [PF_CASES[i] for i in ci]
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    with tempfile.TemporaryDirectory() as d:
        ps = [ctx.Process(target=_peer_worker.run_pipefusion, args=(g, world, port, cases, d)) for g in range(world)]
        [p.start() for p in ps]; [p.join(60) for p in ps]
        print("alive:", [p.is_alive() for p in ps]); [p.kill() for p in ps if p.is_alive()]
        for g in range(world):
            f = os.path.join(d, f"rank{g}.json")
            print(g, open(f).read()[:2000] if os.path.exists(f) else "no result")
