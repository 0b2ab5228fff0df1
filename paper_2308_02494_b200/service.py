"""HTTP + WebSocket rendering service over the device renderer (reference
service.py:1-254).

Same endpoints, request model and semantics as the reference service, so its clients (the viewer,
scripts) switch over unchanged:

  GET  /api/models        artifacts under the served directory (volumes, .apmg models, manifests)
  POST /api/load          {"path": ...} -> the artifact's meta (404 unknown, 400 missing path)
  GET  /api/meta          meta of the loaded artifact (409 before a load)
  POST /api/render        RenderRequest -> PNG bytes, byte-identical to render_frame + PNG encoding
  WS   /api/progressive   one JSON message per progressive pass (base64 PNG); a newer request on
                          the socket or on the same session id cancels the stream at the next pass
                          boundary with {"request_id", "cancelled": true}
  GET  /api/stats         last frame time and field-query throughput

Frames come from this package's renderer (render.py: device rays, tensor-core field queries,
front-to-back compositing); the service is plumbing.  Renders run in a worker thread (anyio), one
progressive pass per hop, so the event loop keeps reading the socket between passes.
"""
from __future__ import annotations

import asyncio
import base64
import json
import time
from dataclasses import dataclass, field as dc_field
from pathlib import Path

import anyio.to_thread
from fastapi import FastAPI, HTTPException, Response, WebSocket, WebSocketDisconnect
from pydantic import BaseModel, ValidationError

from .decomposition import DecomposedField
from .model import load_model
from .render import (Camera, ModelField, RenderConfig, TransferFunction, VolumeField, image_to_png_bytes,
                     render_frame, render_progressive)
from .volume import load_header, load_volume

DEFAULT_PORT = 8080


class RenderRequest(BaseModel):
    """Body of /api/render and of each /api/progressive message (service.py:45-52)."""
    camera: dict
    tf: dict | None = None
    samples_per_ray: int = 128
    batch_size: int = 65536
    progressive: bool = False
    request_id: str = ""
    session_id: str = "default"

    def inputs(self):
        """(camera, transfer function, render config); invalid parameters -> HTTP 400."""
        try:
            return (Camera.from_json(self.camera),
                    TransferFunction.from_json(self.tf) if self.tf else TransferFunction(),
                    RenderConfig(samples_per_ray=self.samples_per_ray, batch_size=self.batch_size))
        except Exception as exc:  # noqa: BLE001 -- any construction error is a bad request
            raise HTTPException(status_code=400, detail=f"invalid render request: {exc}") from exc


def _artifact_kind(path: Path) -> str | None:
    if path.name == "manifest.json":
        return "decomposed"
    if path.suffix == ".apmg":
        return "model"
    if path.suffix == ".json" and path.with_suffix(".raw").exists():
        try:
            obj = json.loads(path.read_text())
        except (OSError, ValueError):
            return None
        if isinstance(obj, dict) and "dims" in obj:
            return "volume"
    return None


def list_artifacts(root: Path) -> list[dict]:
    """Loadable artifacts under `root`, sorted by path (service.py:62-82)."""
    out = []
    for path in sorted(root.rglob("*")):
        kind = _artifact_kind(path)
        if kind:
            out.append({"path": str(path.relative_to(root)), "kind": kind})
    return out


def open_artifact(root: Path, rel: str):
    """(field, meta) of an artifact path relative to `root` (service.py:85-115); anything outside
    the served directory or of an unknown type is a 404."""
    target = (root / rel).resolve()
    if not target.is_relative_to(root.resolve()) or not target.exists():
        raise HTTPException(status_code=404, detail=f"unknown artifact: {rel}")
    kind = _artifact_kind(target)
    if kind == "decomposed":
        fld = DecomposedField.load(target)
        plan = fld.manifest.plan
        return fld, {"kind": kind, "path": rel, "dims": list(fld.manifest.volume_header.dims), "vmin": fld.vmin,
                     "vmax": fld.vmax, "bricks": list(plan.counts), "ghost": plan.ghost}
    if kind == "model":
        fld = ModelField(load_model(target))
        return fld, {"kind": kind, "path": rel, "dims": None, "vmin": fld.vmin, "vmax": fld.vmax, "bricks": None}
    if kind == "volume":
        vol = load_volume(target.with_suffix(".raw"), load_header(target))
        fld = VolumeField(vol)
        return fld, {"kind": kind, "path": rel, "dims": list(vol.dims), "vmin": fld.vmin, "vmax": fld.vmax,
                     "bricks": None}
    raise HTTPException(status_code=404, detail=f"unknown artifact type: {rel}")


@dataclass
class ServiceState:
    """Loaded artifact, frame statistics and the render generation of every session id: bumping a
    session's generation supersedes its in-flight progressive stream."""
    root: Path
    field: object = None
    meta: dict | None = None
    stats: dict = dc_field(default_factory=lambda: {"last_frame_ms": None, "points_per_sec": None})
    sessions: dict = dc_field(default_factory=dict)

    def require_field(self):
        if self.field is None:
            raise HTTPException(status_code=409, detail="no artifact loaded")
        return self.field

    def record(self, seconds: float, points: int) -> None:
        self.stats = {"last_frame_ms": seconds * 1e3, "points_per_sec": points / seconds if seconds > 0 else None}

    def begin(self, session_id: str) -> int:
        gen = self.sessions.get(session_id, 0) + 1
        self.sessions[session_id] = gen
        return gen


async def _progressive_stream(state: ServiceState, ws: WebSocket, inbox: asyncio.Queue, req: RenderRequest,
                              generation: int):
    """Send one message per pass until the final pass or a superseding request (checked only at
    pass boundaries, service.py:216-254); returns the next queued message (None: socket closed)."""
    camera, tf, cfg = req.inputs()
    passes = render_progressive(state.field, camera, tf, cfg)
    done = object()
    t0, points = time.perf_counter(), 0
    while True:
        item = await anyio.to_thread.run_sync(next, passes, done)
        if item is done:
            break
        points += item.samples_evaluated
        await ws.send_json({"request_id": req.request_id, "pass_index": item.index, "level": item.level,
                            "final": item.final,
                            "png": base64.b64encode(image_to_png_bytes(item.preview)).decode("ascii")})
        if item.final:
            break
        if state.sessions.get(req.session_id, 0) != generation or not inbox.empty():
            await ws.send_json({"request_id": req.request_id, "cancelled": True})
            return await inbox.get()
    state.record(time.perf_counter() - t0, points)
    return await inbox.get()


def create_app(artifact_dir, viewer_dir=None) -> FastAPI:
    """The service over the artifacts in `artifact_dir` (+ the static viewer, if given)."""
    app = FastAPI(title="apmg-b200 renderer service")
    state = ServiceState(root=Path(artifact_dir))
    app.state.svc = state  # the loaded field is app.state.svc.field

    @app.get("/api/models")
    def models():
        return {"models": list_artifacts(state.root)}

    @app.post("/api/load")
    def load(body: dict):
        rel = body.get("path")
        if not rel:
            raise HTTPException(status_code=400, detail="missing 'path'")
        state.field, state.meta = open_artifact(state.root, rel)
        return state.meta

    @app.get("/api/meta")
    def meta():
        state.require_field()
        return state.meta

    @app.get("/api/stats")
    def stats():
        return state.stats

    @app.post("/api/render")
    async def render(req: RenderRequest):
        fld = state.require_field()
        camera, tf, cfg = req.inputs()
        t0 = time.perf_counter()
        image = await anyio.to_thread.run_sync(render_frame, fld, camera, tf, cfg)
        state.record(time.perf_counter() - t0, camera.width * camera.height * cfg.samples_per_ray)
        return Response(content=image_to_png_bytes(image), media_type="image/png")

    @app.websocket("/api/progressive")
    async def progressive(ws: WebSocket):
        await ws.accept()
        inbox: asyncio.Queue = asyncio.Queue()

        async def pump():  # every incoming message queues; a queued message supersedes a stream
            try:
                while True:
                    await inbox.put(await ws.receive_text())
            except WebSocketDisconnect:
                await inbox.put(None)

        reader = asyncio.create_task(pump())
        try:
            msg = await inbox.get()
            while msg is not None:
                try:
                    req = RenderRequest(**json.loads(msg))
                except (ValueError, ValidationError) as exc:
                    await ws.send_json({"error": f"invalid request: {exc}"})
                    msg = await inbox.get()
                    continue
                if state.field is None:
                    await ws.send_json({"error": "no artifact loaded", "request_id": req.request_id})
                    msg = await inbox.get()
                    continue
                try:
                    req.inputs()
                except HTTPException as exc:
                    await ws.send_json({"error": exc.detail, "request_id": req.request_id})
                    msg = await inbox.get()
                    continue
                msg = await _progressive_stream(state, ws, inbox, req, state.begin(req.session_id))
        except WebSocketDisconnect:
            pass
        finally:
            reader.cancel()

    if viewer_dir is not None and Path(viewer_dir).exists():
        from fastapi.staticfiles import StaticFiles
        app.mount("/", StaticFiles(directory=str(viewer_dir), html=True), name="viewer")
    return app


def serve(artifact_dir, host: str = "127.0.0.1", port: int = DEFAULT_PORT, viewer_dir=None) -> None:
    import uvicorn
    uvicorn.run(create_app(artifact_dir, viewer_dir), host=host, port=port)
