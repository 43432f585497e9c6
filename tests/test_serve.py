"""HTTP serving on the GPU path (serve.py), following the reference's
tests/test_server.py: endpoints, status codes, determinism, and concurrent
requests (each on its own engine + stream) equal to serial ones."""

import base64
import json
import threading
from concurrent.futures import ThreadPoolExecutor
from http.client import HTTPConnection

import numpy as np
import pytest

from conftest import random_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def server():
    from paper_2507_07136_b200.io import QuerySet
    from paper_2507_07136_b200.projection import CameraPose
    from paper_2507_07136_b200.query import QueryEmbedding
    from paper_2507_07136_b200.serve import ServeSession, make_server
    rng = np.random.default_rng(11)
    scene = random_scene(rng, num_gaussians=400, num_levels=2, L=8, K=2, D=8)
    qs = QuerySet(dim=8, canonicals=rng.standard_normal((4, 8)),
                  queries=[QueryEmbedding(f"class{c}", rng.standard_normal(8)) for c in range(4)])
    pose = CameraPose.from_dict({"position": [0.4, 0.3, -3.4], "look_at": [0, 0, 0], "fov_y_deg": 42.0,
                                 "width": 24, "height": 24})
    session = ServeSession(scene, qs, size_cap=128, default_pose=pose, engines=3)
    srv = make_server(session, host="127.0.0.1", port=0)
    t = threading.Thread(target=srv.serve_forever, daemon=True)
    t.start()
    yield srv.server_address
    srv.shutdown()
    srv.server_close()


def request(addr, method, path, body=None, raw=None):
    conn = HTTPConnection(addr[0], addr[1], timeout=60)
    payload = raw if raw is not None else (json.dumps(body) if body is not None else None)
    conn.request(method, path, body=payload, headers={"Content-Type": "application/json"} if payload else {})
    resp = conn.getresponse()
    out = (resp.status, dict(resp.getheaders()), resp.read())
    conn.close()
    return out


def pose_doc():
    return {"position": [0.4, 0.3, -3.4], "look_at": [0, 0, 0], "fov_y_deg": 42.0}


def qbody(**kw):
    b = {"camera": pose_doc(), "width": 24, "height": 24, "query": "class0", "level": "auto", "window": 3}
    b.update(kw)
    return b


def test_meta_and_unknown_endpoint(server):
    status, headers, data = request(server, "GET", "/meta")
    doc = json.loads(data)
    assert status == 200 and doc["L"] == 8 and doc["K"] == 2 and doc["levels"] == 2
    assert doc["queries"] == [f"class{c}" for c in range(4)]
    assert doc["request_id"].startswith("req-") and "X-Request-Id" in headers
    assert request(server, "GET", "/nope")[0] == 404


def test_render_png_and_errors(server):
    status, headers, a = request(server, "POST", "/render", {"camera": pose_doc(), "width": 32, "height": 32})
    assert status == 200 and headers["Content-Type"] == "image/png" and a[:8] == b"\x89PNG\r\n\x1a\n"
    _, _, b = request(server, "POST", "/render", {"camera": pose_doc(), "width": 32, "height": 32})
    assert a == b
    status, _, data = request(server, "POST", "/render", {"camera": pose_doc(), "width": 4096, "height": 4096})
    assert status == 413 and "exceeds" in json.loads(data)["error"]
    status, _, data = request(server, "POST", "/render", raw="{oops")
    assert status == 400 and "malformed JSON" in json.loads(data)["error"]
    assert request(server, "POST", "/render", {"width": 16, "height": 16})[0] == 400


def test_query_fields_and_errors(server):
    status, _, data = request(server, "POST", "/query", qbody())
    doc = json.loads(data)
    assert status == 200
    for k in ("query", "level", "timings_ms", "point", "score_stats", "settings", "overlay_png_base64"):
        assert k in doc
    assert base64.b64decode(doc["overlay_png_base64"])[:8] == b"\x89PNG\r\n\x1a\n"
    explicit = json.loads(request(server, "POST", "/query", qbody(level=doc["level"]))[2])
    assert explicit["point"] == doc["point"]
    status, _, data = request(server, "POST", "/query", qbody(query="sofa"))
    assert status == 404 and json.loads(data)["available"] == [f"class{c}" for c in range(4)]
    assert request(server, "POST", "/query", qbody(query=[0.1] * 8))[0] == 200
    assert request(server, "POST", "/query", qbody(query=[0.1] * 7))[0] == 400
    assert request(server, "POST", "/query", qbody(level=5))[0] == 400
    assert request(server, "POST", "/query", qbody(window=4))[0] == 400


def test_concurrent_requests_match_serial(server):
    bodies = [qbody(query=f"class{c % 4}", width=16 + 4 * (c % 3)) for c in range(12)]
    serial = [json.loads(request(server, "POST", "/query", b)[2]) for b in bodies]
    with ThreadPoolExecutor(max_workers=6) as pool:
        conc = list(pool.map(lambda b: json.loads(request(server, "POST", "/query", b)[2]), bodies))
    for s, c in zip(serial, conc):
        for k in ("level", "point", "score_stats", "overlay_png_base64"):
            assert s[k] == c[k], k
